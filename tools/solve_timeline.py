"""Per-launch device times of one mds_solve (profiled launches) on a C3 step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mdsgen
import paper_2605_13736_b200 as mds
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
prob = mdsgen.config_problem(cfg)
st = mds.KKTStep(mds.DeviceProblem(prob))
st.run(); torch.cuda.synchronize()
for rep in range(3):
    mds.profile_begin(); st.run(); mds.profile_end()
    tl = mds.profile_timeline()
    sol = [(c, s, e) for c, s, e in tl if c.startswith("solve") or c == "recover"]
    t0 = sol[0][1]
    print(" ".join(f"{c}[{(s - t0) * 1e3:.0f},{(e - t0) * 1e3:.0f}]" for c, s, e in sol))
