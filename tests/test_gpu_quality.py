"""Eigenpair quality through the C ABI (the paper's Fig. 3b metrics, PAPER.md:253-258;
SURVEY 8(f) NEXT-3): pairwise eigenvector angles, L2 reconstruction error
||M y - lambda y|| against the fp64 matrix, reorthogonalisation on vs off, and the
device residual estimate |beta_{m+1} s_{m,k}| against the measured residual
(they agree to rounding)."""
import numpy as np
import pytest

import synthgen as S
from bench import eigen_quality

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3s():
    return S.config_matrix("C3S")


def _solve(A, K, storage, reorth):
    import paper_2201_07498_b200 as T
    vs = storage
    with T.TopkEig(A, K, storage=storage, compute="f64", values_storage=vs, m=K, reorth=reorth) as h:
        return h.solve(seed=3, vectors=True, vec_dtype="f64")


@pytest.mark.parametrize("storage,dot_tol,est_tol", [("f64", 1e-10, 1e-10), ("f32", 1e-5, 1e-5)])
def test_quality_reorth_on(c3s, storage, dot_tol, est_tol):
    r = _solve(c3s, 24, storage, 1)
    kf = len(r.eigenvectors)
    assert kf == 24
    q = eigen_quality(c3s, r.eigenvectors, r.eigenvalues[:kf])
    assert q["max_abs_dot"] <= dot_tol, q
    assert q["mean_angle_deg"] > 90.0 - 1e-3
    # the device residual estimate is the measured residual (values stored in the
    # same dtype as the vectors, so M here is the exact input matrix only for f64;
    # for f32 the input weights k/128 are exact in f32 as well)
    est = np.asarray(r.residual_est[:kf])
    assert np.max(np.abs(est - q["residuals"])) <= est_tol * abs(r.eigenvalues[0])


def test_quality_reorth_off_is_not_better(c3s):
    on = eigen_quality(c3s, *(lambda r: (r.eigenvectors, r.eigenvalues[:len(r.eigenvectors)]))(_solve(c3s, 24, "f64", 1)))
    off_r = _solve(c3s, 24, "f64", -1)
    off = eigen_quality(c3s, off_r.eigenvectors, off_r.eigenvalues[:len(off_r.eigenvectors)])
    assert abs(90.0 - off["mean_angle_deg"]) >= abs(90.0 - on["mean_angle_deg"]) - 1e-9
    assert off["max_abs_dot"] >= on["max_abs_dot"] - 1e-12
