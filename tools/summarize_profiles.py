"""Turn the raw ncu outputs of tools/profile_round.sh (gpurun_out/) into the
committed summaries under profiles/:
  launches_<tag>.csv          the ncu --metrics gpu__time_duration.sum launch list (copied)
  launches_<tag>_summary.csv  per kernel: launches and us per step, share of the step
  ncu_<name>_<tag>.csv        key metrics of each --set full capture (one row per kernel)
usage: python tools/summarize_profiles.py <tag> [steps_in_launch_list]"""
import csv
import os
import re
import shutil
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 9
src, dst = "gpurun_out", "profiles"

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread"]


def short(name):
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", name)
    name = re.sub(r"^void ", "", name)
    return re.sub(r"\(.*$", "", name).replace("(int)", "").replace("(bool)", "")


def launch_summary():
    path = os.path.join(src, "launches.csv")
    if not os.path.exists(path):
        return
    shutil.copy(path, os.path.join(dst, f"launches_{tag}.csv"))
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "nsecond"
        us = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
        k = short(r[ik])
        tot[k] += us
        cnt[k] += 1
    total = sum(tot.values())
    with open(os.path.join(dst, f"launches_{tag}_summary.csv"), "w") as f:
        f.write(f"# per step (the launch list holds {steps} eager steps); ncu-serialised cold-cache times\n")
        f.write("kernel,launches_per_step,us_per_step,share\n")
        for k in sorted(tot, key=lambda k: -tot[k]):
            f.write(f"{k},{cnt[k] / steps:.1f},{tot[k] / steps:.1f},{tot[k] / total:.4f}\n")


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "second": 1e6}


def norm(v, unit):
    """ncu --page raw values carry per-metric units (bytes in byte/Kbyte/Mbyte/..., times in
    nsecond/usecond/...): normalise bytes to bytes and times to microseconds."""
    v = v.replace(",", "")
    if unit in SCALE and v:
        try:
            return f"{float(v) * SCALE[unit]:.6g}"
        except ValueError:
            return v
    return v


def full_summary(rep, out):
    path = os.path.join(src, rep)
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    body = [r for r in rows[2:] if len(r) == len(hdr)]
    unit_of = dict(zip(hdr, units))
    cols = [k + (" [bytes]" if unit_of.get(k, "").endswith("byte") else (" [us]" if unit_of.get(k, "").endswith("second")
                                                                         else "")) for k in KEYS]
    with open(os.path.join(dst, out), "w") as f:
        f.write("kernel," + ",".join(cols) + "\n")
        for r in body:
            d = dict(zip(hdr, r))
            f.write(short(d.get("Kernel Name", "?")).replace(",", ";") + "," +
                    ",".join(norm(d.get(k, ""), unit_of.get(k, "")) for k in KEYS) + "\n")


launch_summary()
for rep, out in [("upd_full_raw.csv", f"ncu_k_update_tma_{tag}.csv"), ("misc_full_raw.csv", f"ncu_misc_{tag}.csv"),
                 ("exact_full_raw.csv", f"ncu_k_panel_exact_{tag}.csv"),
                 ("solve_full_raw.csv", f"ncu_solve_vectors_{tag}.csv"),
                 ("cond_full_raw.csv", f"ncu_condense_{tag}.csv"), ("batched_full_raw.csv", f"ncu_batched_{tag}.csv"),
                 ("ipm_full_raw.csv", f"ncu_ipm_{tag}.csv")]:
    full_summary(rep, out)
print("\n".join(sorted(os.listdir(dst))))
