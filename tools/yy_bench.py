"""Time mds_condense alone on C3 (events), for kernel experiments."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mdsgen
import paper_2605_13736_b200 as mds
prob = mdsgen.config_problem("C3")
dp = mds.DeviceProblem(prob); st = mds.KKTStep(dp)
def run():
    mds.condense(dp.plan, dp.val, dp.h_ss, dp.sigma_s, dp.H_dd, dp.ldh, dp.sigma_d, dp.J_d, dp.ldj, dp.d_h,
                 dp.delta_w, dp.delta_c, dp.r, st.M, st.ldm, st.rhs, st.w, st.status)
for _ in range(3): run()
torch.cuda.synchronize()
mds.profile_begin()
for _ in range(5): run()
prof = mds.profile_end()
print({k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items() if v[1]})
