"""HostPipeline (step.py): Newton steps from pinned HOST inputs with the copies
overlapped with compute give bitwise the results of the device-resident step
(the same kernels on the same inputs), for every step of a sequence, and the
oracle's inertia / solution (Eq.(5)-(6))."""
import numpy as np
import pytest

import mdsgen
import oracle
from tests.helpers import rel_inf

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_13736_b200 as mds  # noqa: E402


@pytest.mark.parametrize("use_graph", [True, False])
def test_pipeline_matches_device_step_and_oracle(use_graph):
    prob = mdsgen.config_problem("C2")
    sv = mdsgen.step_vectors_for(prob, seed=3)
    st = mds.KKTStep(mds.DeviceProblem(prob), sv=sv)
    st.run()
    ref = st.results()
    pipe = mds.HostPipeline(prob, sv=sv, use_graph=use_graph)
    host = pipe.pinned_inputs()
    hout = pipe.pinned_outputs()
    for steps in (1, 4):
        for h in hout:
            h.zero_()
        pipe.run(steps, host, hout)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(hout[0].numpy(), ref["dxy"])
        assert tuple(int(v) for v in hout[1]) == ref["inertia"] == prob.expected_inertia
        np.testing.assert_array_equal(hout[2].numpy(), ref["dx_s"])
        assert hout[3][0].item() == ref["vec"]["alpha_p"]
    o = oracle.newton_step(prob)
    assert rel_inf(hout[0].numpy(), o["dxy"]) <= 1e-8


def test_pipeline_sees_new_host_inputs():
    # the second step's inputs differ (delta-free rescaled r): its result must follow them
    prob = mdsgen.config_problem("C1")
    pipe = mds.HostPipeline(prob, use_graph=True)
    host = pipe.pinned_inputs()
    hout = pipe.pinned_outputs()
    pipe.run(1, host, hout)
    torch.cuda.synchronize()
    x1 = hout[0].clone()
    host[mds.HostPipeline.IN.index("r")].mul_(2.0)
    pipe.run(3, host, hout)
    torch.cuda.synchronize()
    np.testing.assert_allclose(hout[0].numpy(), 2.0 * x1.numpy(), rtol=1e-12, atol=0)
