"""Where an IPM iteration's time goes (C3-shaped QP): wall per iteration, the
inertia-checked Newton step (events), and per-class device time of one profiled
trajectory (profiled launches are serialised by their events).
usage: python tools/ipm_prof.py [C3|C2]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdsgen  # noqa: E402
import paper_2605_13736_b200 as mds  # noqa: E402
from paper_2605_13736_b200.ipm import IPMSolver  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
qp = mdsgen.qp_config(cfg)
s = IPMSolver(qp, use_graph=os.environ.get("GRAPH", "1") == "1")
s.solve()
s.reset(qp)
torch.cuda.synchronize()
t = time.perf_counter()
r = s.solve()
torch.cuda.synchronize()
wall = (time.perf_counter() - t) * 1e3
its = max(r["iterations"], 1)
print(f"{cfg}: {its} iterations, {wall:.1f} ms wall = {wall / its:.2f} ms/iter; newton mean "
      f"{sum(r['newton_ms']) / len(r['newton_ms']):.2f} ms")
s.reset(qp)
mds.profile_begin()
r = s.solve()
prof = mds.profile_end()
print({k: (round(v[0] / its, 3), round(v[1] / its, 1)) for k, v in prof.items() if v[1]})
