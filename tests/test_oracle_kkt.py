"""O8 K2 mat-vec of the full Eq.(5) matrix against a
brute-force dense K assembled entry by entry from the block definition, and the
defining property of the step: K [dx_s; dx_d; dy] = r for the oracle's Newton
step (condense -> BK -> solve -> recover), i.e. the compression is exact."""
import numpy as np

import mdsgen
import oracle


def dense_K(q):
    n_s, n_d, m_E, m_I = q.n_s, q.n_d, q.m_E, q.m_I
    m = m_E + m_I
    Nf = n_s + n_d + m
    K = np.zeros((Nf, Nf))
    for k in range(n_s):
        K[k, k] = q.h_ss[k] + q.sigma_s[k] + q.delta_w
        for t in range(q.rowptr[k], q.rowptr[k + 1]):
            c = q.colidx[t]
            K[k, n_s + n_d + c] = q.val[t]
            K[n_s + n_d + c, k] = q.val[t]
    H = np.asarray(q.H_dd)
    for i in range(n_d):
        for j in range(n_d):
            K[n_s + i, n_s + j] = H[max(i, j), min(i, j)]
        K[n_s + i, n_s + i] += q.sigma_d[i] + q.delta_w
    Jd = np.asarray(q.J_d)
    for c in range(m):
        for j in range(n_d):
            K[n_s + n_d + c, n_s + j] = Jd[c, j]
            K[n_s + j, n_s + n_d + c] = Jd[c, j]
        K[n_s + n_d + c, n_s + n_d + c] = -((1.0 / q.d_h[c - m_E]) if c >= m_E else 0.0) - q.delta_c
    return K


def test_matvec_vs_dense_entrywise():
    for shape, dw, dc in [((60, 7, 3, 4), 0.0, 0.0), ((150, 10, 5, 0), 0.3, 1e-3), ((0, 6, 2, 2), 0.0, 0.5),
                          ((80, 0, 4, 5), 0.1, 0.0)]:
        q = mdsgen.g1_quasidefinite(*shape, seed=sum(shape), delta_w=dw, delta_c=dc)
        x = np.random.default_rng(3).standard_normal(q.n_s + q.n_d + q.m_E + q.m_I)
        ref = dense_K(q) @ x
        got = oracle.kkt_matvec(q, x)
        assert np.abs(got - ref).max() <= 1e-13 * max(np.abs(ref).max(), 1.0)


def test_newton_step_solves_full_system():
    q = mdsgen.g1_quasidefinite(2000, 40, 20, 20, seed=8)
    st = oracle.newton_step(q)
    x = np.concatenate([st["dx_s"], st["dxy"]])
    r = np.asarray(q.r)
    assert np.abs(oracle.kkt_matvec(q, x) - r).max() <= 1e-11 * np.abs(r).max()
    # mutation: a wrong sign in one block is caught
    x2 = x.copy()
    x2[q.n_s + 3] *= -1.0
    assert np.abs(oracle.kkt_matvec(q, x2) - r).max() > 1e-6
