"""Thick-restart Lanczos (reading Q26) through the
C ABI against oracle.solve_thick_restart on the same seeded inputs: the same
restart count and step count, Ritz values of the final basis normwise within the
north-star tolerances (1e-8 DDD, 1e-4 mixed), eigenvectors within 1e-5, the
convergence-driven stop at the same cycle, and loopback parts = one part."""
import numpy as np
import pytest

import oracle as O
import synthgen as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import paper_2201_07498_b200 as T
    return T


@pytest.fixture(scope="module")
def c3s():
    return S.config_matrix("C3S")


def _normwise(a, b):
    a, b = np.sort(a), np.sort(b)
    return np.abs(a - b).max() / np.abs(b).max()


def _vectors_close(res, ref, tol):
    th = ref.theta_all
    for k in range(len(ref.eigenvalues)):
        t = ref.eigenvalues[k]
        gap = np.min(np.abs(np.delete(th, np.argmin(np.abs(th - t))) - t)) / abs(ref.eigenvalues[0])
        if gap < 1e-4:
            continue
        y, yr = res.eigenvectors[k].astype(np.float64), ref.eigenvectors[k]
        assert abs(np.linalg.norm(y) - 1) < 1e-6
        d = min(np.linalg.norm(y - yr), np.linalg.norm(y + yr))
        assert d <= tol * max(1.0, 1e-4 / gap), (k, d, gap)


@pytest.mark.parametrize("storage,tol", [("f64", 1e-8), ("f32", 1e-4)])
def test_thick_restart_matches_oracle(T, c3s, storage, tol):
    K, m, keep, R, seed = 16, 48, 24, 3, 5
    ref = O.solve_thick_restart(c3s.rowptr, c3s.col, c3s.val, K, m, keep, R, seed=seed, tau=O.TAU[storage])
    with T.TopkEig(c3s, K, storage=storage, compute="f64", m=m, restart_keep=keep, max_restarts=R) as h:
        res = h.solve(seed=seed, vectors=True)
        _, _, th = h.tridiag()
    assert res.info["restarts"] == ref.extra["restarts"] == R
    assert res.info["iterations"] == ref.extra["iterations"] == m + R * (m - keep)
    assert res.info["k_found"] == K and res.info["breakdown"] == 0
    assert _normwise(th, ref.theta_all) <= tol
    err = np.abs(res.eigenvalues - ref.eigenvalues).max() / abs(ref.eigenvalues[0])
    assert err <= tol
    _vectors_close(res, ref, 1e-5 if storage == "f64" else 1e-3)
    # beta_{m+1} of the last cycle (reading Q6), read at the cycle's own step count
    bref = ref.lanczos.beta[ref.lanczos.m_found]
    assert abs(res.info["beta_next"] - bref) <= tol * abs(ref.eigenvalues[0]), (res.info["beta_next"], bref)


def test_thick_restart_converged_stop(T, c3s):
    K, m, keep, tol, seed = 16, 48, 24, 1e-6, 5
    ref = O.solve_thick_restart(c3s.rowptr, c3s.col, c3s.val, K, m, keep, 40, tol=tol, seed=seed)
    assert ref.extra["restarts"] < 40
    with T.TopkEig(c3s, K, "f64", "f64", m=m, restart_keep=keep, max_restarts=40, conv_tol=tol) as h:
        res = h.solve(seed=seed, vectors=True)
    assert res.info["restarts"] == ref.extra["restarts"]
    assert res.info["iterations"] == ref.extra["iterations"]
    assert res.info["converged_stop"] == 1
    assert np.all(res.residual_est <= tol * abs(res.eigenvalues[0]) * (1 + 1e-12))
    assert np.abs(res.eigenvalues - ref.eigenvalues).max() <= 1e-8 * abs(ref.eigenvalues[0])
    # the converged pairs are eigenpairs of M: explicit residual within the tolerance
    import scipy.sparse as sp
    M = sp.csr_matrix((c3s.val, c3s.col, c3s.rowptr), shape=(c3s.n, c3s.n))
    for k in range(K):
        y = res.eigenvectors[k]
        assert np.linalg.norm(M @ y - res.eigenvalues[k] * y) <= 2 * tol * abs(res.eigenvalues[0])


def test_thick_restart_loopback_parts(T, c3s):
    out = []
    for G in (1, 3):
        with T.TopkEig(c3s, 16, "f64", "f64", m=40, restart_keep=20, max_restarts=2, parts=G) as h:
            out.append(h.solve(seed=9, vectors=False))
    assert out[0].info["iterations"] == out[1].info["iterations"]
    assert np.abs(out[0].eigenvalues - out[1].eigenvalues).max() <= 1e-10 * abs(out[0].eigenvalues[0])


def test_thick_restart_deterministic_and_graph(T, c3s):
    with T.TopkEig(c3s, 8, "f32", "f64", m=32, restart_keep=12, max_restarts=2) as h:
        a = h.solve(seed=3)
        b = h.solve(seed=3)
    with T.TopkEig(c3s, 8, "f32", "f64", m=32, restart_keep=12, max_restarts=2, use_graph=False) as h:
        c = h.solve(seed=3)
    assert np.array_equal(a.eigenvalues, b.eigenvalues) and np.array_equal(a.eigenvectors, b.eigenvectors)
    assert np.array_equal(a.eigenvalues, c.eigenvalues)
