"""SCOPF scenario batch on one GPU: concurrent-stream graph replays give the
same per-scenario results as running each scenario alone, and match the CPU
oracle (inertia exact, solution within the north-star tolerance)."""
import numpy as np
import pytest

import mdsgen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_13736_b200 as mds  # noqa: E402
from paper_2605_13736_b200 import scopf  # noqa: E402


def test_scopf_batch_matches_single_and_oracle():
    base = mdsgen.scopf_base(seed=5, n_s=6000, n_d=100, m_E=40, m_I=60)
    fn = lambda s: mdsgen.scopf_scenario(base, s, seed=5)
    svf = lambda p, s: mdsgen.step_vectors_for(p, seed=100 + s)
    ids = scopf.partition(9, 2, 1)          # this "rank" owns 1, 3, 5, 7
    batch = scopf.ScopfBatch(base, fn, ids, svf)
    for _ in range(2):
        batch.newton_step()
    torch.cuda.synchronize()
    stats = batch.stop_test()
    assert stats["n_scenarios"] == len(ids) and stats["n_bad_inertia"] == 0
    recs = scopf.gather_records(batch.records, 9)
    assert list(recs[:, 0]) == ids
    for i, s in enumerate(ids):
        p = fn(s)
        # the same scenario alone (a batch of one): bitwise the same (no cross-scenario arithmetic,
        # so P = 1, 2, 4, 8 ranks give identical per-scenario records)
        one = mds.BatchedKKTStep([p], plan=batch.plan, svs=[svf(p, s)])
        one.run()
        a = one.results(0)
        b = batch.results(i)
        np.testing.assert_array_equal(a["dxy"], b["dxy"])
        assert a["inertia"] == b["inertia"] == p.expected_inertia
        assert recs[i, 4] == b["vec"]["alpha_p"] and recs[i, 5] == b["vec"]["alpha_d"]
        ref = oracle.newton_step(p)
        assert np.abs(b["dxy"] - ref["dxy"]).max() <= 1e-8 * np.abs(ref["dxy"]).max()
