"""The seeded input generators (mdsgen): the torch-built G3 used at the C5 size
(N = 32768, 8.6 GB, impractical in numpy) must be the numpy G3 (same draws,
same reflectors), and its inertia must be the closed form (eigvalsh)."""
import numpy as np
import pytest

import mdsgen

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("N,n2,seed", [(300, 40, 5), (257, 100, 11)])
def test_g3_torch_equals_numpy(N, n2, seed):
    A, ine = mdsgen.g3_prescribed(N, seed=seed, n2x2=n2)
    B, ine2 = mdsgen.g3_prescribed_torch(N, seed=seed, n2x2=n2, device="cpu")
    assert ine == ine2
    assert np.abs(A - B.numpy()).max() <= 1e-12 * np.abs(A).max()
    ev = np.linalg.eigvalsh(B.numpy())
    assert (int((ev > 0).sum()), 0, int((ev < 0).sum())) == ine2
