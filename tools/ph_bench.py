"""Time the pivot-heavy factor + solve (bench.pivot_heavy_block) with more steps.
usage: python tools/ph_bench.py [N] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
r = bench.pivot_heavy_block(N, steps, torch.device("cuda", 0))
print(N, round(r["ms"], 3), r["exact_bk_columns"], r["inertia_ok"])
