"""Debug helper: factor one G1 instance through the C-ABI and compare with the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mdsgen, oracle
import paper_2605_13736_b200 as mds
shape = tuple(int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (2000, 64, 40, 26)))
prob = mdsgen.g1_quasidefinite(*shape, seed=3)
st = mds.KKTStep(mds.DeviceProblem(prob))
ine = st.run(sync_inertia=True)
torch.cuda.synchronize()
out = st.results()
ref = oracle.newton_step(prob)
print("inertia", ine, ref["inertia"], "status", out["status"],
      "relerr", np.abs(out["dxy"] - ref["dxy"]).max() / np.abs(ref["dxy"]).max())
