#!/usr/bin/env python
"""bench.py — one Newton step of the condensed-KKT hot path (§2:
condense Eq.(5)->(6), Bunch-Kaufman LDL^T with inertia, solves + dx_s
recovery, barrier vector kernels) on synthetic OPF-shaped MDS inputs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

N=1 workload: BASELINE.json configs[2] "C3" (ACOPF-shaped, n_d+m = 8192,
n_s = 1M) — the config the north star's FP64 target (N >= 8192) is quoted on.
Multi-GPU: `--gpus N` re-launches itself as N ranks (torch.distributed.run,
NCCL) unless already under a launcher.  C3 is one KKT system per Newton step
and does not shard (BK needs a global pivot search per column), so ranks run
independent replicas; value = steps of all ranks /
max-rank time.  The same line carries a "scopf" block: the sharded workload of
the north star, C4's 256 SCOPF scenarios strong-scaled over the N ranks
(round-robin, one batched graph per rank, NCCL only for the per-step stopping
test), value = scenario Newton steps/s of the whole job.

--impl reference: the CPU oracle (oracle/, plain C, OpenMP over all host
cores, bit-identical to one thread) on the same workload: the full step when
it fits a 45 s budget, else a leading-block sample extrapolated and flagged
"projected": true (see cpu_baseline.sample).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "condensed-KKT factor+solve/s, FP64 TFLOP/s vs peak; Newton iters/s"
UNIT = "newton_iters/s"
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peaks_r01.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=3072, help="oracle factor sample size (leading block)")
    ap.add_argument("--scenarios", type=int, default=256, help="C4: total SCOPF scenarios (strong scaling)")
    ap.add_argument("--no-scopf", action="store_true", help="C3: skip the C4 scenario-batch block")
    ap.add_argument("--no-ipm", action="store_true", help="C3: skip the IPM-trajectory block")
    ap.add_argument("--ipm-sweep", default="2000,8000,10000", help="nlpMDS_ex4 sizes k for the IPM block")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        # nvidia-smi can take a second or more to start: wait for its first sample
        # (up to 10 s) so the timed region is covered
        t0 = time.time()
        while self.p is not None and time.time() - t0 < 10.0:
            if os.path.getsize(self.f.name) > 0 or self.p.poll() is not None:
                break
            time.sleep(0.05)
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.15)   # one more sample after the timed region
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                self.p.wait()
        self.f.flush()

    def summary(self):
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def update_traffic():
    """DRAM bytes (read + write) of the one k_update_tma launch captured with ncu --set full
    (profiles/ncu_k_update_tma_r02.csv, C3 panel 10: trailing order n2 = 7488; r01 as fallback)
    and that launch's algorithmic bytes (C lower read + written once, L21 and W21 read once)."""
    import csv
    n2 = 7488
    alg = 2 * 8 * n2 * (n2 + 1) / 2 + 2 * 8 * n2 * 64
    for tag, cols, scale in (("r02", ("dram__bytes_read.sum [bytes]", "dram__bytes_write.sum [bytes]"), 1.0),
                             ("r01", ("dram__bytes_read.sum", "dram__bytes_write.sum"), 1e6)):
        path = os.path.join(ROOT, "profiles", f"ncu_k_update_tma_{tag}.csv")
        try:
            rows = list(csv.reader(open(path)))
            d = dict(zip(rows[0], rows[1]))
            b = (float(d[cols[0]]) + float(d[cols[1]])) * scale
            return b, {"source": f"profiles/ncu_k_update_tma_{tag}.csv", "launch": "C3 panel 10, n2 = 7488",
                       "dram_bytes": b, "algorithmic_bytes": alg, "ratio": b / alg}
        except Exception:
            continue
    return None, None


def fp64_peak():
    try:
        d = json.load(open(FP64_PEAK_FILE))
        dm = max(m["tflops"] for m in d["micro"] if m["kernel"].startswith("dmma"))
        return dm, d.get("cublas_dgemm_8192_burst_tflops")
    except Exception:
        return 37.2, None


def measured_hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def algorithmic(prob, panels):
    """Algorithmic work of one step at this instance."""
    n_s, n_d, m, nnz, N = prob.n_s, prob.n_d, prob.m, prob.nnz, prob.N
    condense_bytes = (12 * nnz + 4 * (n_s + 1) + 16 * n_s + 8 * n_d * (n_d + 1) // 2 + 8 * m * n_d + 8 * n_d
                      + 8 * prob.m_I + 8 * (n_s + N) + 8 * N + 8 * N * (N + 1) // 2 + 8 * n_s)
    # trailing-update flops from the actual panel boundaries: sum n2 (n2+1) kb
    upd = 0
    ends = list(panels[1:]) + [N]
    for s, e in zip(panels, ends):
        n2 = int(N) - int(e)
        upd += n2 * (n2 + 1) * (int(e) - int(s))
    factor_flops = N ** 3 / 3.0
    solve_flops = 2.0 * N * N
    solve_bytes = 8 * N * N + 8 * 6 * N + 12 * nnz + 40 * n_s
    return dict(condense_bytes=condense_bytes, update_flops=float(upd), factor_flops=factor_flops,
                solve_flops=solve_flops, solve_bytes=solve_bytes)


# ----------------------------------------------------------------------------- CPU oracle
FULL_STEP_BUDGET_S = 45.0   # run the full oracle step when its projection fits this budget


def oracle_full_step(prob, sv):
    """The oracle's whole Newton step, unextrapolated: condensation, BK factor of the
    full N x N M (OpenMP over independent trailing-update columns: bit-identical to one
    thread), inertia, solve, recovery, step vectors.  Returns (seconds, detail)."""
    import oracle
    t0 = time.perf_counter()
    M, rhs, w = oracle.condense(prob)
    t1 = time.perf_counter()
    LD, ipiv, _ = oracle.bk_factor(M)
    t2 = time.perf_counter()
    tol = oracle.default_tol(M)
    ine = oracle.inertia(LD, ipiv, tol)
    x = oracle.bk_solve(LD, ipiv, rhs, tol)
    del LD
    dxs = oracle.recover(prob, w, prob.r[:prob.n_s], x[prob.n_d:])
    dx = np.concatenate([dxs, x[:prob.n_d]])
    oracle.step_vectors(sv.x, dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    oracle.norm_inf(prob.r)
    t3 = time.perf_counter()
    return t3 - t0, dict(t_condense=t1 - t0, t_factor=t2 - t1, t_rest=t3 - t2, inertia=ine)


def oracle_sample(prob, sv, ns_factor, reps=1):
    """The oracle on one step of this workload, on all host cores.  If the full step's
    projection (from a timed leading-block factorization) fits FULL_STEP_BUDGET_S, the
    full step is executed (projected = False); otherwise the leading ns x ns block is
    factored and the factor / solve times are extrapolated (projected = True).
    Returns (seconds per step, detail)."""
    import oracle
    nth = oracle.num_threads()
    cpu_model = ""
    try:
        with open("/proc/cpuinfo") as f:
            cpu_model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    N = prob.N
    ns = min(ns_factor, N)
    t0 = time.perf_counter()
    M, rhs, w = oracle.condense(prob)
    t_cond = time.perf_counter() - t0
    A = np.asfortranarray(M[:ns, :ns])
    t0 = time.perf_counter()
    LD, ipiv, _ = oracle.bk_factor(A)
    t_fac = time.perf_counter() - t0
    t0 = time.perf_counter()
    tol = oracle.default_tol(A)
    oracle.bk_solve(LD, ipiv, rhs[:ns], tol)
    t_sol = time.perf_counter() - t0
    del M, LD
    t0 = time.perf_counter()
    dxs = oracle.recover(prob, w, prob.r[:prob.n_s], np.zeros(prob.m))
    dx = np.concatenate([dxs, np.zeros(prob.n_d)])
    oracle.step_vectors(sv.x, dx, sv.lo, sv.up, sv.zl, sv.zu, sv.dzl, sv.dzu, sv.tau, sv.mu)
    oracle.norm_inf(prob.r)
    t_vec = time.perf_counter() - t0
    proj = t_cond + t_fac * (N / ns) ** 3 + t_sol * (N / ns) ** 2 + t_vec
    base = dict(cores=nth, cpu_model=cpu_model, host_cpus=os.cpu_count())
    if ns == N or proj <= FULL_STEP_BUDGET_S:
        t, det = (t_cond + t_fac + t_sol + t_vec, {}) if ns == N else oracle_full_step(prob, sv)
        sample = (f"oracle (plain C, OpenMP {nth} threads on {cpu_model or 'host CPU'}) executing the FULL step: "
                  f"condensation of all {prob.n_s} sparse variables, BK factor + solve of the full {N}x{N} M, "
                  f"recovery, step vectors ({t:.1f} s measured, not projected)")
        return t, dict(base, projected=False, sample=sample, **det)
    sample = (f"oracle (plain C, OpenMP {nth} threads on {cpu_model or 'host CPU'}): full condensation + recovery + "
              f"step vectors, BK factor+solve of the leading {ns}x{ns} block of M extrapolated x(N/{ns})^3 (factor) "
              f"and x(N/{ns})^2 (solve) -- PROJECTED (full step projected at {proj:.0f} s > "
              f"{FULL_STEP_BUDGET_S:.0f} s budget); measured {t_cond + t_fac + t_sol + t_vec:.2f} s of CPU work")
    return proj, dict(base, projected=True, sample=sample, t_condense=t_cond, t_factor_sample=t_fac,
                      t_solve_sample=t_sol, t_vec=t_vec, ns=ns)


def run_reference_c5(args):
    import mdsgen
    import oracle
    N = 32768
    ns = min(args.ref_sample, 2048)
    A, _ = mdsgen.g3_prescribed(ns, seed=5005)   # same family, bounded size (the 8.6 GB matrix is GPU-generated)
    projs = []
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        LD, ipiv, _ = oracle.bk_factor(A)
        tf = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.bk_solve(LD, ipiv, np.ones(ns), oracle.default_tol(A))
        ts = time.perf_counter() - t0
        projs.append(tf * (N / ns) ** 3 + ts * (N / ns) ** 2)
    t_step = float(np.mean(projs))
    val = 1.0 / t_step
    nth = oracle.num_threads()
    sample = (f"oracle (plain C, OpenMP {nth} threads) BK factor+solve of a {ns}x{ns} G3 matrix, extrapolated "
              f"x(N/{ns})^3 / x(N/{ns})^2 to N={N} -- PROJECTED")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "factor_solve/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C5 " + CONFIG_DESC["C5"], "N": N},
            "projected": True,
            "cpu_baseline": {"value": val, "unit": "factor_solve/s", "cores": nth, "kind": "oracle", "sample": sample,
                             "projected": True},
            "e2e": {"value": val, "unit": "factor_solve/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": time.perf_counter() - wall0}
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    import mdsgen
    if rank != 0:
        return
    if args.config == "C5":
        run_reference_c5(args)
        return
    prob = mdsgen.config_problem(args.config)
    sv = mdsgen.step_vectors_for(prob, seed=7)
    # one probe decides full vs projected; warm-up = the probe (page-in, thread pool)
    t_probe, det = oracle_sample(prob, sv, args.ref_sample)
    steps = args.steps
    ts = []
    wall0 = time.perf_counter()
    if det["projected"]:
        for _ in range(steps):
            t, det = oracle_sample(prob, sv, args.ref_sample)
            ts.append(t)
    else:
        # full steps, bounded to ~3 minutes of CPU work in total (the count executed is reported)
        steps = max(1, min(args.steps, int(180.0 / max(t_probe, 1e-3))))
        for _ in range(steps):
            t, _d = oracle_full_step(prob, sv) if prob.N > args.ref_sample else oracle_sample(prob, sv, args.ref_sample)
            ts.append(t)
    wall = time.perf_counter() - wall0
    t_step = float(np.mean(ts))
    val = 1.0 / t_step
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": 1, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} " + CONFIG_DESC[args.config], "N": prob.N, "n_s": prob.n_s,
                       "nnz": prob.nnz},
            "projected": bool(det["projected"]), "steps_requested": args.steps,
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": det["cores"], "kind": "oracle",
                             "sample": det["sample"], "projected": bool(det["projected"]),
                             "cpu_model": det["cpu_model"]},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


CONFIG_DESC = {
    "C1": "toy MDS n_s=400, n_d=20, m=20 (N=40), one Newton step",
    "C2": "synthetic MDS N=n_d+m=1024, n_s=100k, CSR J_s ~5 nnz/row, one Newton step",
    "C3": "ACOPF-shaped MDS N=n_d+m=8192 (n_d=4096, m_E=m_I=2048), n_s=1M, ~5 nnz/row, one Newton step",
    "C4": "SCOPF scenario N=2048, n_s=131072 (single scenario)",
    "C5": "dense prescribed-spectrum symmetric indefinite N=n_d+m=32768 (8.6 GB), FP64 LDL^T factor+solve stress",
}


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist

    import mdsgen
    import paper_2605_13736_b200 as mds

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    prob = mdsgen.config_problem(args.config)
    sv = mdsgen.step_vectors_for(prob, seed=7)
    dp = mds.DeviceProblem(prob)
    st = mds.KKTStep(dp, sv=sv)
    launches0 = mds.launch_count()
    st.run()
    torch.cuda.synchronize()
    launches_per_step = mds.launch_count() - launches0
    out0 = st.results()
    if out0["status"] != 0 or out0["inertia"] != prob.expected_inertia:
        raise SystemExit(f"bench: step failed status={out0['status']} inertia={out0['inertia']}")
    panels = mds.factor_panels(st.fwork, prob.N)
    alg = algorithmic(prob, panels)

    use_graph = not args.no_graph
    graph = st.capture() if use_graph else None
    stream = torch.cuda.current_stream()

    def step():
        if graph is not None:
            graph.replay()
        else:
            st.run()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # working set (M + the step's inputs) below ~2x L2: flush L2 between timed steps (a 256 MB
    # write, outside the per-step events) so every step starts cold, as in the large configs
    small = 8 * prob.N * prob.N + dp.host_bytes() < 2 * 126e6
    flush_buf = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev) if small else None
    ev_pairs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.steps)] if small else None
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for i in range(args.steps):
            if small:
                flush_buf.fill_(float(i))
                ev_pairs[i][0].record(stream)
            step()
            if small:
                ev_pairs[i][1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1) if not small else sum(a.elapsed_time(b) for a, b in ev_pairs)
    clocks = clk.summary()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * args.steps / (ms_max / 1e3)

    # wall-clock phase times (events between the four C-ABI calls, eager, median of 3)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ph = []
    for _ in range(3):
        st.run(marks=marks)
        torch.cuda.synchronize()
        ph.append([marks[i].elapsed_time(marks[i + 1]) for i in range(4)])
    ph = np.median(np.array(ph), axis=0)
    wall = dict(condense=float(ph[0]), factor=float(ph[1]), solve=float(ph[2]), vectors=float(ph[3]))

    # profiled eager pass: per-kernel-class device time (CUDA events on the launch stream)
    mds.profile_begin()
    st.run()
    prof = mds.profile_end()
    st.check_status()
    tot = sum(v[0] for v in prof.values())
    fac_ms = sum(prof[c][0] for c in ("anorm", "panel_diag", "panel_trsm", "panel_store", "panel_exact", "update",
                                      "finalize"))
    sol_ms = sum(prof[c][0] for c in ("solve_gather", "solve_fwd", "solve_d", "solve_bwd", "solve_scatter",
                                      "recover"))
    cond_ms = sum(prof[c][0] for c in ("condense_rows", "condense_diag", "condense_norm", "condense_tiles"))
    dom = max(prof, key=lambda c: prof[c][0])
    peak_dmma, peak_cublas = fp64_peak()
    hbm, hbm_src = measured_hbm()
    upd_ms, upd_n = prof["update"]
    if dom == "update":
        ach = alg["update_flops"] / (upd_ms * 1e-3) / 1e12
        tb, tnote = update_traffic()
        roof = {"kernel": "k_update (DMMA trailing update)", "bound": "tensor", "achieved": ach, "peak": peak_dmma,
                "unit": "TFLOP/s", "frac": ach / peak_dmma, "traffic": tb, "traffic_note": tnote,
                "peak_source": "measured FP64 DMMA ceiling, profiles/fp64_peaks_r01.json (cuBLAS DGEMM "
                               f"{peak_cublas:.2f} TF/s); MEASURED_PEAKS.json has no FP64 entry",
                "launches": upd_n, "avg_launch_us": upd_ms * 1e3 / max(upd_n, 1)}
    else:
        roof = {"kernel": dom, "bound": "latency", "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": None, "launches": prof[dom][1], "ms": prof[dom][0]}
    kern = {c: {"ms": round(v[0], 4), "launches": v[1], "share": round(v[0] / tot, 4) if tot else 0}
            for c, v in prof.items() if v[1]}

    # end-to-end through the public API with HOST buffers (pinned), copies inside the timed region:
    # mds.HostPipeline uploads every step's inputs and downloads its results on a copy stream,
    # overlapped with the neighbouring steps' compute (two device input sets)
    e2e = None
    if not args.no_e2e:
        pipe = mds.HostPipeline(prob, sv=sv, use_graph=use_graph)
        host = pipe.pinned_inputs()
        hout = pipe.pinned_outputs()
        h2d, d2h = pipe.bytes_per_step(host, hout)
        pipe.run(2, host, hout)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pipe.run(args.steps, host, hout, start=f0, end=f1)
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ine_h = tuple(int(v) for v in hout[1])
        if ine_h != prob.expected_inertia:
            raise SystemExit(f"bench: e2e step inertia {ine_h}")
        e2e = {"value": world * args.steps / (float(te.item()) / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "api": "paper_2605_13736_b200.HostPipeline (copies of step i+1 / i-1 "
               "overlapped with step i on a copy stream)"}
        del pipe

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        t_or, det = oracle_sample(prob, sv, args.ref_sample)
        cpu = {"value": 1.0 / t_or, "unit": UNIT, "cores": det["cores"], "kind": "oracle", "sample": det["sample"],
               "projected": bool(det["projected"]), "cpu_model": det["cpu_model"]}

    if rank == 0:
        fs_ms = fac_ms + sol_ms
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{args.config} " + CONFIG_DESC[args.config], "N": prob.N, "n_s": prob.n_s,
                           "nnz": prob.nnz, "parallelism": f"replicas{world}" if world > 1 else "single",
                           "l2": ("L2 flushed between timed steps (256 MB write outside the per-step events; "
                                  "working set %.0f MB)" % ((8 * prob.N * prob.N + dp.host_bytes()) / 1e6)) if small
                           else "inputs larger than L2 (M alone is %.0f MB)" % (8 * prob.N * prob.N / 1e6),
                           "cuda_graph": use_graph},
                "gpu_launches": launches_per_step * args.steps,
                "roofline": roof,
                "factor_solve_per_s": 1e3 / (wall["factor"] + wall["solve"]),
                "factor_solve_fp64_tflops": (alg["factor_flops"] + alg["solve_flops"]) /
                                            ((wall["factor"] + wall["solve"]) * 1e-3) / 1e12,
                "factor_fp64_tflops": alg["factor_flops"] / (wall["factor"] * 1e-3) / 1e12,
                "factor_fp64_frac_of_peak": alg["factor_flops"] / (wall["factor"] * 1e-3) / 1e12 / peak_dmma,
                "condense_gbs": alg["condense_bytes"] / (wall["condense"] * 1e-3) / 1e9,
                "condense_frac_of_hbm": alg["condense_bytes"] / (wall["condense"] * 1e-3) / 1e9 / hbm,
                "solve_gbs": alg["solve_bytes"] / (wall["solve"] * 1e-3) / 1e9,
                # K1 barrier vectors: 8 FP64 inputs + sigma out per (x_s, x_d) component, plus the
                # residual vector's inf-norm read (~72 B per bounded component)
                "vectors_gbs": (72 * (prob.n_s + prob.n_d) + 8 * (prob.n_s + prob.N)) /
                               (prof["vectors"][0] * 1e-3) / 1e9 if prof["vectors"][0] > 0 else None,
                "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src,
                "phase_ms_wall": wall,
                "phase_ms_kernel_sum": {"condense": cond_ms, "factor": fac_ms, "solve": sol_ms,
                                        "vectors": prof["vectors"][0]},
                "kernels": kern, "panels": int(len(panels)),
                "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
                "inertia": list(out0["inertia"])}
        return line
    return None


def run_scopf(args, rank, world, emit=True):
    """C4: SCOPF scenario batch, scenarios round-robin over ranks; per Newton step
    the rank's whole local batch as ONE graph of batched launches + ONE small NCCL
    all-reduce pair for the global stopping test (read on the host)."""
    import torch
    import torch.distributed as dist

    import mdsgen
    import paper_2605_13736_b200 as mds
    from paper_2605_13736_b200 import scopf

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    base = mdsgen.scopf_base()
    fn = lambda s_: mdsgen.scopf_scenario(base, s_)
    svf = lambda p_, s_: mdsgen.step_vectors_for(p_, seed=100 + s_)
    ids = scopf.partition(args.scenarios, world, rank)
    t0 = time.time()
    batch = scopf.ScopfBatch(base, fn, ids, svf)
    setup_s = time.time() - t0
    for _ in range(args.warmup):
        batch.newton_step()
        batch.stop_test()
    torch.cuda.synchronize()
    # library launches per Newton step (the graph replays exactly this sequence)
    l1 = mds.launch_count()
    batch.bt.run()
    torch.cuda.synchronize()
    per_step = mds.launch_count() - l1
    mds.profile_begin()
    batch.bt.run()
    prof = mds.profile_end()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            batch.newton_step()
            st = batch.stop_test()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # end to end: every step uploads the local batch's inputs from pinned host memory and
    # downloads its results (directions, inertias, step-vector scalars); copies not overlapped
    e2e = None
    if not args.no_e2e:
        bt = batch.bt
        ins = [bt.val, bt.h_ss, bt.sigma_s, bt.H_dd, bt.sigma_d, bt.J_d, bt.d_h, bt.r]
        host = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True).copy_(x.cpu()) for x in ins]
        outs = [bt.dirn, bt.inertia] + ([bt.vout] if bt.sv is not None else [])
        hout = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in outs]
        h2d = sum(x.numel() * x.element_size() for x in host)
        d2h = sum(x.numel() * x.element_size() for x in hout)

        def e2e_step():
            for d_, h_ in zip(ins, host):
                d_.copy_(h_, non_blocking=True)
            batch.newton_step()
            for h_, d_ in zip(hout, outs):
                h_.copy_(d_, non_blocking=True)
            return batch.stop_test()

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": args.scenarios * args.steps / (float(te.item()) / 1e3), "unit": "scenario_newton_iters/s",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
               "note": "per step the whole batch's inputs cross PCIe (~25 MB per scenario), not overlapped"}
        del host, hout
    recs = scopf.gather_records(batch.records, args.scenarios)
    value = args.scenarios * args.steps / (ms_max / 1e3)
    if rank == 0:
        N = base.N
        nloc = len(ids)
        fl = args.scenarios * args.steps * (N ** 3 / 3.0 + 2.0 * N * N)
        upd_ms, upd_n = prof["update"]
        # trailing-update flops of the local batch per step: sum over panels of n2 (n2+1) kb, kb = 64
        upd_fl = 0.0
        k = 0
        while k < N:
            kb = min(64, N - k)
            n2 = N - k - kb
            upd_fl += n2 * (n2 + 1) * kb
            k += kb
        upd_fl *= nloc
        line = {"metric": METRIC, "value": value, "unit": "scenario_newton_iters/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": "C4 " + f"SCOPF {args.scenarios} contingency scenarios, N=2048 each "
                           "(n_d=1024, m_E=m_I=512, n_s=131072, shared pattern), round-robin over ranks, "
                           "batched C-ABI (one graph of batched launches per rank)",
                           "N": N, "scenarios": args.scenarios, "parallelism": f"scenario-dp{world}",
                           "cuda_graph": True, "l2": "inputs larger than L2 (8.6 GB of M per 256 scenarios)"},
                "gpu_launches": per_step * args.steps,
                "factor_solve_fp64_tflops_aggregate": fl / (ms_max * 1e-3) / 1e12,
                "roofline": {"kernel": "k_update_tma<5> (batched DMMA trailing update)", "bound": "tensor",
                             "achieved": upd_fl / (upd_ms * 1e-3) / 1e12, "peak": fp64_peak()[0],
                             "unit": "TFLOP/s", "frac": upd_fl / (upd_ms * 1e-3) / 1e12 / fp64_peak()[0],
                             "traffic": None, "launches": upd_n, "avg_launch_us": upd_ms / max(upd_n, 1) * 1e3},
                "factor_solve_frac_of_peak": fl / (ms_max * 1e-3) / 1e12 / world / fp64_peak()[0],
                "kernels": {c: {"ms": round(v[0], 4), "launches": v[1]} for c, v in prof.items() if v[1]},
                "stop_test": st, "records_gathered": int(recs.shape[0]),
                "all_inertia_ok": bool(st["n_bad_inertia"] == 0), "setup_s": setup_s,
                "clocks": clk.summary(), "e2e": e2e, "cpu_baseline": None}
        if emit:
            print(json.dumps(line), flush=True)
        return line
    return None


def run_ipm(args, rank, world):
    """NEXT-2: a whole interior-point trajectory on the C3-shaped convex QP (n_s = 1M,
    N = 8192; mdsgen.qp_config), every Newton iteration through the hot path + the IPM
    vector kernels (paper_2605_13736_b200.ipm, R23), to e_0 <= 1e-8.  One
    untimed trajectory first (page-in, attributes), then a timed one from the same start."""
    import torch

    import mdsgen
    from paper_2605_13736_b200.ipm import IPMSolver

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    t0 = time.time()
    qp = mdsgen.qp_config(args.config)
    setup_s = time.time() - t0
    sol = IPMSolver(qp)
    sol.solve()          # untimed: page-in, attributes, graph capture
    sol.reset(qp)
    e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        torch.cuda.synchronize()
        e0_.record()
        res = sol.solve()
        e1_.record()
        torch.cuda.synchronize()
    ms = e0_.elapsed_time(e1_)
    h = res["history"]
    its = max(res["iterations"], 1)
    return {"workload": f"{args.config}-shaped convex QP (n_s={qp.base.n_s}, n_d={qp.base.n_d}, m_E={qp.base.m_E}, "
                        f"m_I={qp.base.m_I}, N={qp.base.N}), filter line-search IPM to e_0 <= 1e-8",
            "status": res["status"], "iterations": res["iterations"], "e0": res["e0"], "final_mu": res["mu"],
            "trajectory_ms": ms, "newton_iters_per_s": its / (ms / 1e3),
            "newton_step_ms_mean": float(np.mean(res["newton_ms"])) if res["newton_ms"] else None,
            "line_search_trials": int(sum(r["trials"] for r in h)),
            "iterations_with_delta_w": int(sum(r["delta_w"] > 0 for r in h)),
            "exact_bk_columns_total": int(sum(r["exact_cols"] for r in h)),
            "exact_bk_columns_max": int(max((r["exact_cols"] for r in h), default=0)),
            "interchanges_total": int(sum(r["swaps"] for r in h)),
            "inertia_ok_every_iteration": bool(all(r["inertia"] == (qp.base.n_d, 0, qp.base.m) for r in h)),
            "host_syncs_per_iteration": "inertia (24 B), error norms, line-search scalars, factor counters",
            "setup_s": setup_s, "clocks": clk.summary(),
            "paper_sweep": ipm_paper_sweep(args)}


def ipm_paper_sweep(args):
    """The paper's own workload: the nlpMDS_ex4 mini-app problem (
    mdsgen.synthetic_problem, compressed size N = 2k+3) solved to e_0 <= 1e-8 by the device
    IPM at k = 2000 / 8000 / 10000 (N = 4003 / 16003 / 20003: the paper's "matrix size
    16,000" and "20,000").  Per-iteration times are context against the paper's V100
    numbers (MAGMA 4.49 s per iteration at 16,000), not a target."""
    import torch

    import mdsgen
    from paper_2605_13736_b200.ipm import IPMSolver

    out = []
    for k in [int(v) for v in args.ipm_sweep.split(",") if v]:
        qp = mdsgen.synthetic_problem(k)
        sol = IPMSolver(qp)
        sol.solve()      # untimed: page-in, graph capture
        sol.reset(qp)
        torch.cuda.synchronize()
        e0_, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0_.record()
        res = sol.solve()
        e1_.record()
        torch.cuda.synchronize()
        ms = e0_.elapsed_time(e1_)
        its = max(res["iterations"], 1)
        x = sol.solution()["x"]
        out.append({"k": k, "N": qp.base.N, "status": res["status"], "iterations": res["iterations"],
                    "e0": res["e0"], "ms_per_iteration": ms / its,
                    "newton_step_ms_mean": float(np.mean(res["newton_ms"])) if res["newton_ms"] else None,
                    "newton_step_fp64_frac_of_peak": ((qp.base.N ** 3 / 3.0) / (float(np.mean(res["newton_ms"])) * 1e-3)
                                                      / 1e12 / fp64_peak()[0]) if res["newton_ms"] else None,
                    "max_abs_x_minus_closed_form": float(np.abs(x - 0.5).max()),
                    "paper_context": ("V100 MAGMA 4.49 s / iteration at matrix size 16,000 (P:541)" if k == 8000 else
                                      ("V100 peak 4.2 TF/s at 20,000 (P:634)" if k == 10000 else None))})
        del sol
        torch.cuda.empty_cache()
    return out


def pivot_heavy_block(N, steps, dev):
    """The C3-sized Newton matrix when Bunch-Kaufman has to pivot: factor + solve of the
    N x N G3 matrix (prescribed spectrum, N/8 2x2 blocks, random orthogonal mixing:
    the speculative panels fail and the exact BK columns run), timed like C5 (M restored
    outside the events).  Context for the C3 line, whose quasi-definite matrix never
    leaves the fast path."""
    import torch

    import mdsgen
    import paper_2605_13736_b200 as mds

    A, ine = mdsgen.g3_prescribed_torch(N, seed=3003, device=dev)
    A0 = A.T.contiguous().reshape(-1)
    del A
    M = torch.empty_like(A0)
    piv = torch.empty(2 * N, dtype=torch.int32, device=dev)
    ine_d = torch.zeros(3, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device=dev)
    swork = torch.empty(mds.solve_workspace_size(N), dtype=torch.uint8, device=dev)
    b = torch.as_tensor(np.random.default_rng(N).standard_normal(N), dtype=torch.float64, device=dev)
    x = torch.empty(N, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def fs():
        mds.factor(N, M, N, piv, -1.0, ine_d, status, fwork, sync=False)
        mds.solve(None, N, M, N, piv, b, None, None, None, x, None, -1.0, fwork, status, swork)

    M.copy_(A0)
    fs()
    torch.cuda.synchronize()
    got = tuple(int(v) for v in ine_d.cpu())
    stats = mds.factor_stats(fwork)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for e0, e1 in evs:
        M.copy_(A0)
        e0.record(stream)
        fs()
        e1.record(stream)
    torch.cuda.synchronize()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs) / steps
    return {"workload": f"G3 prescribed-spectrum N={N} ({N // 8} 2x2 blocks, orthogonally mixed), factor + solve",
            "ms": ms, "factor_solve_per_s": 1e3 / ms, "fp64_frac_of_peak": (N ** 3 / 3.0) / (ms * 1e-3) / 1e12
            / fp64_peak()[0], "inertia_ok": got == tuple(ine) and int(status.item()) == 0,
            "panels": int(stats[0]), "interchanges": int(stats[1]), "exact_bk_columns": int(stats[2])}


def run_c5(args, rank, world):
    """C5 stress: factor + solve of the N = 32768 G3 matrix (8.6 GB) per step (replicas under torchrun).
    M is restored from a device copy before every step, outside the timed region (CUDA events bracket
    exactly mds_factor + mds_solve)."""
    import torch
    import torch.distributed as dist

    import mdsgen
    import paper_2605_13736_b200 as mds

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    N = 32768
    A, ine = mdsgen.g3_prescribed_torch(N, seed=5005, device=dev)
    A0 = A.T.contiguous().reshape(-1)          # column-major copy of the input
    del A
    M = torch.empty_like(A0)
    piv = torch.empty(2 * N, dtype=torch.int32, device=dev)
    ine_d = torch.zeros(3, dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device=dev)
    swork = torch.empty(mds.solve_workspace_size(N), dtype=torch.uint8, device=dev)
    b = torch.as_tensor(np.random.default_rng(N).standard_normal(N), dtype=torch.float64, device=dev)
    x = torch.empty(N, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def fs():
        mds.factor(N, M, N, piv, -1.0, ine_d, status, fwork, sync=False)
        mds.solve(None, N, M, N, piv, b, None, None, None, x, None, -1.0, fwork, status, swork)

    launches0 = mds.launch_count()
    M.copy_(A0)
    fs()
    torch.cuda.synchronize()
    launches_per_step = mds.launch_count() - launches0
    got = tuple(int(v) for v in ine_d.cpu())
    if int(status.item()) != 0 or got != ine:
        raise SystemExit(f"bench C5: status={int(status.item())} inertia={got} expected={ine}")
    for _ in range(max(args.warmup - 1, 0)):
        M.copy_(A0)
        fs()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(dev.index) as clk:
        for e0, e1 in evs:
            M.copy_(A0)
            e0.record(stream)
            fs()
            e1.record(stream)
        torch.cuda.synchronize()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    clocks = clk.summary()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * args.steps / (ms_max / 1e3)
    flops = N ** 3 / 3.0 + 2.0 * N * N
    # profiled pass: update-kernel share and its achieved FP64 rate
    M.copy_(A0)
    mds.profile_begin()
    fs()
    prof = mds.profile_end()
    panels = mds.factor_panels(fwork, N)
    upd = 0
    ends = list(panels[1:]) + [N]
    for s0, e in zip(panels, ends):
        n2 = N - int(e)
        upd += n2 * (n2 + 1) * (int(e) - int(s0))
    peak_dmma, peak_cublas = fp64_peak()
    upd_ms, upd_n = prof["update"]
    ach = upd / (upd_ms * 1e-3) / 1e12
    roof = {"kernel": "k_update (DMMA trailing update)", "bound": "tensor", "achieved": ach, "peak": peak_dmma,
            "unit": "TFLOP/s", "frac": ach / peak_dmma, "traffic": None,
            "peak_source": "measured FP64 DMMA ceiling, profiles/fp64_peaks_r01.json", "launches": upd_n}
    # end to end: the matrix from pinned host memory, x back
    e2e = None
    if not args.no_e2e:
        hA = torch.empty(A0.shape, dtype=A0.dtype, pin_memory=True).copy_(A0.cpu())
        hx = torch.empty(N, dtype=torch.float64, pin_memory=True)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            M.copy_(hA, non_blocking=True)
            fs()
            hx.copy_(x, non_blocking=True)
        f1.record(stream)
        torch.cuda.synchronize()
        e2e = {"value": args.steps / (f0.elapsed_time(f1) / 1e3) * world, "unit": "factor_solve/s",
               "h2d_bytes_per_step": int(hA.numel() * 8), "d2h_bytes_per_step": int(N * 8)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle
        ns = min(args.ref_sample, 2048)
        Ah = A0.reshape(N, N)[:ns, :ns].cpu().numpy().T.copy(order="F")
        t0 = time.perf_counter()
        LD, ipiv, _ = oracle.bk_factor(Ah)
        tf = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.bk_solve(LD, ipiv, np.ones(ns), oracle.default_tol(Ah))
        tsol = time.perf_counter() - t0
        proj = tf * (N / ns) ** 3 + tsol * (N / ns) ** 2
        cpu = {"value": 1.0 / proj, "unit": "factor_solve/s", "cores": oracle.num_threads(), "kind": "oracle",
               "projected": True,
               "sample": f"oracle (plain C, OpenMP {oracle.num_threads()} threads) BK factor+solve of the leading "
                         f"{ns}x{ns} block, extrapolated x(N/{ns})^3 / x(N/{ns})^2 -- PROJECTED; measured "
                         f"{tf + tsol:.2f} s"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "factor_solve/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "C5 " + CONFIG_DESC["C5"], "N": N, "parallelism": "replicas" if world > 1 else "single",
                           "l2": "inputs larger than L2 (M is 8.6 GB)", "cuda_graph": False},
                "gpu_launches": launches_per_step * args.steps, "roofline": roof,
                "factor_solve_fp64_tflops": flops / (ms_step * 1e-3) / 1e12,
                "factor_solve_frac_of_peak": flops / (ms_step * 1e-3) / 1e12 / peak_dmma,
                "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu, "inertia": list(got),
                "kernels_ms": {c: round(v[0], 3) for c, v in prof.items() if v[1]},
                "panels": len(panels)}
        print(json.dumps(line), flush=True)


def spawn(args):
    """`python bench.py --gpus N` outside a launcher: re-run this script as N ranks
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1, NCCL)."""
    import socket
    s_ = socket.socket()
    s_.bind(("127.0.0.1", 0))
    port = s_.getsockname()[1]
    s_.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "WARN")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    if args.config == "C4":
        run_scopf(args, rank, world)
    elif args.config == "C5":
        run_c5(args, rank, world)
    else:
        line = run_ours(args, rank, world)
        if args.config == "C3" and not args.no_scopf:
            # the sharded workload of the north star, measured in the same run: C4's scenario batch
            # strong-scaled over the same ranks (scenarios round-robin, NCCL only for the stopping test)
            import torch
            torch.cuda.empty_cache()
            sc = run_scopf(args, rank, world, emit=False)
            if rank == 0 and line is not None and sc is not None:
                line["scopf"] = {k: sc[k] for k in ("value", "unit", "n_gpus", "ms_per_step", "scaling",
                                                    "gpu_launches", "factor_solve_fp64_tflops_aggregate",
                                                    "factor_solve_frac_of_peak", "all_inertia_ok", "roofline",
                                                    "clocks", "e2e")}
                line["scopf"]["workload"] = sc["config"]["workload"]
                line["scopf"]["collectives_per_step"] = "1 MAX + 1 SUM all_reduce of 5 + 2 doubles (NCCL)"
        if args.config == "C3" and not args.no_ipm and rank == 0 and line is not None:
            import torch
            torch.cuda.empty_cache()
            line["ipm"] = run_ipm(args, rank, world)
        if args.config == "C3" and not args.no_ipm and rank == 0 and line is not None:
            import torch
            torch.cuda.empty_cache()
            line["pivot_heavy"] = pivot_heavy_block(8192, 3, torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
        if rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
