import sys, os
sys.path.insert(0, os.getcwd())
import torch, mdsgen
from paper_2605_13736_b200.ipm import IPMSolver
s = IPMSolver(mdsgen.qp_config("C3"), use_graph=False)
for _ in range(3):
    s._k0(s.xy, s.Kxy)
torch.cuda.synchronize()
