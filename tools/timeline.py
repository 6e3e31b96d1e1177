"""Per-panel critical-path analysis of one C3 factorization (profiled launches)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mdsgen
import paper_2605_13736_b200 as mds
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
prob = mdsgen.config_problem(cfg)
st = mds.KKTStep(mds.DeviceProblem(prob))
st.run(); torch.cuda.synchronize()
mds.profile_begin(); st.run(); mds.profile_end()
tl = mds.profile_timeline()
t0 = min(t[1] for t in tl)
out = [(c, s - t0, e - t0) for c, s, e in tl]
json.dump(out, open("gpurun_out/timeline.json", "w"))
# per-panel: diag start -> next diag start, and what ran
diag = [i for i, t in enumerate(out) if t[0] == "panel_diag"]
rows = []
for k in range(len(diag) - 1):
    seg = out[diag[k]:diag[k + 1]]
    per = {}
    for c, s, e in seg:
        per[c] = per.get(c, 0.0) + (e - s)
    rows.append((k, out[diag[k + 1]][1] - out[diag[k]][1], per))
for k, dur, per in rows[::8]:
    print(k, f"{dur*1e3:.1f}us", {c: round(v * 1e3, 1) for c, v in per.items()})
print("total factor span ms", out[diag[-1]][2] - out[diag[0]][1])
