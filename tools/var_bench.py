"""A/B the factorization's launch-structure variants (mds_set_variant) on one
Newton step: CUDA-graph replay, CUDA events, median of 20.
usage: python tools/var_bench.py [C3|C2|C5] "k=v,k=v" "k=v" ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdsgen  # noqa: E402
import paper_2605_13736_b200 as mds  # noqa: E402

cfg = sys.argv[1]
variants = sys.argv[2:] or [""]
prob = mdsgen.config_problem(cfg)
for var in variants:
    mds.set_variant("default")
    for kv in filter(None, var.split(",")):
        k, v = kv.split("=")
        mds.set_variant(k, int(v))
    st = mds.KKTStep(mds.DeviceProblem(prob))
    g = st.capture()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(20):
        ev[0].record()
        g.replay()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ts.sort()
    out = st.results()
    print(f"{cfg} [{var or 'default'}]: step {ts[10]:.3f} ms (best {ts[0]:.3f}) inertia {out['inertia']} status {out['status']}",
          flush=True)
    del g, st
    torch.cuda.empty_cache()
