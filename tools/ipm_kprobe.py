"""A few IPM iterations (C3 QP, eager) for an ncu launch list of the IPM vector kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mdsgen  # noqa: E402
from paper_2605_13736_b200.ipm import IPMSolver  # noqa: E402

s = IPMSolver(mdsgen.qp_config("C3"), opts=dict(max_iter=3), use_graph=False)
s.solve()
