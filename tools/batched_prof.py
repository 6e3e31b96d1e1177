"""Per-kernel-class time of one batched C4 Newton step (B scenarios, profiled
launches: events around every launch, so concurrency is removed) and the graph
time of the same step.  usage: BATCH=64 python tools/batched_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdsgen  # noqa: E402
import paper_2605_13736_b200 as mds  # noqa: E402

B = int(os.environ.get("BATCH", "64"))
for kv in filter(None, os.environ.get("VARIANTS", "").split(",")):
    k, v = kv.split("=")
    mds.set_variant(k, int(v))
base = mdsgen.scopf_base()
bt = mds.BatchedKKTStep((B, lambda i: (mdsgen.scopf_scenario(base, i), mdsgen.step_vectors_for(base, seed=i))))
bt.run()
torch.cuda.synchronize()
g = bt.capture()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for _ in range(5):
    ev[0].record()
    g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
mds.profile_begin()
bt.run()
torch.cuda.synchronize()
prof = mds.profile_end()
print(os.environ.get("VARIANTS", ""), f"B={B}: graph step {sorted(ts)[2]:.3f} ms;",
      {k: (round(v[0], 3), int(v[1])) for k, v in prof.items() if v[1]})
