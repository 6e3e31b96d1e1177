import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, mdsgen
import paper_2605_13736_b200 as mds
base = mdsgen.scopf_base()
B = int(os.environ.get("OZB", "64"))
bt = mds.BatchedKKTStep((B, lambda i: (mdsgen.scopf_scenario(base, i), None)))
mds.set_variant("ozaki", int(os.environ.get("OZ", "1")))
bt.run(); torch.cuda.synchronize()
bt.run(); torch.cuda.synchronize()
