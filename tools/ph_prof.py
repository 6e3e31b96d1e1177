import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import mdsgen, paper_2605_13736_b200 as mds
N = 8192
dev = torch.device("cuda", 0)
A, ine = mdsgen.g3_prescribed_torch(N, seed=3003, device=dev)
A0 = A.T.contiguous().reshape(-1); del A
M = torch.empty_like(A0)
piv = torch.empty(2 * N, dtype=torch.int32, device=dev)
ine_d = torch.zeros(3, dtype=torch.int64, device=dev)
status = torch.zeros(1, dtype=torch.int32, device=dev)
fwork = torch.empty(mds.factor_workspace_size(N), dtype=torch.uint8, device=dev)
for it in range(2):
    M.copy_(A0); torch.cuda.synchronize()
    if it == 1: mds.profile_begin()
    mds.factor(N, M, N, piv, -1.0, ine_d, status, fwork, sync=False)
    torch.cuda.synchronize()
prof = mds.profile_end()
print({k: (round(v[0], 3), v[1]) for k, v in prof.items() if v[1]})
print(mds.factor_stats(fwork))
