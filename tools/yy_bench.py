"""Time mds_condense alone (CUDA events, L2 flushed between calls) for kernel
experiments: per-kernel-class ms and algorithmic GB/s.
usage: python tools/yy_bench.py [C3|C2|C4] [uniform|local] [nnz_per_row]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdsgen  # noqa: E402
import paper_2605_13736_b200 as mds  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
pattern = sys.argv[2] if len(sys.argv) > 2 else "uniform"
npr = int(sys.argv[3]) if len(sys.argv) > 3 else None
if cfg == "C4":
    prob = mdsgen.scopf_scenario(mdsgen.scopf_base(), 1)
elif npr is not None:
    shp = mdsgen.CONFIGS[cfg]
    prob = mdsgen.g1_quasidefinite(shp["n_s"], shp["n_d"], shp["m_E"], shp["m_I"], 3000, pattern=pattern,
                                   nnz_per_row=npr)
else:
    prob = mdsgen.config_problem(cfg, pattern=pattern)
for kv in filter(None, os.environ.get("VARIANTS", "").split(",")):
    k, v = kv.split("=")
    mds.set_variant(k, int(v))
dp = mds.DeviceProblem(prob)
st = mds.KKTStep(dp)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run():
    mds.condense(dp.plan, dp.val, dp.h_ss, dp.sigma_s, dp.H_dd, dp.ldh, dp.sigma_d, dp.J_d, dp.ldj, dp.d_h,
                 dp.delta_w, dp.delta_c, dp.r, st.M, st.ldm, st.rhs, st.w, st.status, anorm_out=st.anorm,
                 work=st.cwork)


n_s, n_d, m, N, nnz = prob.n_s, prob.n_d, prob.m, prob.N, prob.nnz
alg = (12 * nnz + 4 * (n_s + 1) + 16 * n_s + 8 * n_d * (n_d + 1) // 2 + 8 * m * n_d + 8 * n_d + 8 * prob.m_I
       + 8 * (n_s + N) + 8 * N + 8 * N * (N + 1) // 2 + 8 * n_s)
for _ in range(3):
    run()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(10):
    flush.zero_()
    ev[0].record()
    run()
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
mds.profile_begin()
for _ in range(5):
    flush.zero_()
    run()
prof = mds.profile_end()
ms = sorted(ts)[len(ts) // 2]
print(os.environ.get("VARIANTS", ""), f"{cfg} {pattern} npr={npr} nnz={nnz} pairs={dp.plan.npairs if hasattr(dp.plan, 'npairs') else '?'}: condense {ms:.4f} ms median ({min(ts):.4f} best), algorithmic {alg / 1e6:.1f} MB -> "
      f"{alg / ms / 1e6:.0f} GB/s", {k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items() if v[1]})
