"""SURVEY 8(f) NEXT-4 in the default -m gpu run: ONE part holding more than 2^31
nonzeros (64-bit physical offsets: chunk first nonzero, logical rowptr), with a
closed-form spectrum instead of a slow oracle solve.

M = blockdiag(c_b 1_{s x s}), b = 0..B-1, s = 6554, B = 51, c_b = (64 + b) / 128
(exact in bf16/f32/f64): nnz = B s^2 = 2,190,640,716 > 2^31 in one part (G = 1), every
row a big row of s entries. Each block is rank one, so the nonzero eigenvalues are
exactly lambda_b = c_b s (eigenvector: the block's indicator), the rest 0.
Checks: every sampled SpMV row (y_r = c_b sum_{j in block(r)} x_j) within the rigorous
fp64 bound; the K = 8 Ritz values of the FDF solve (m = 16) each within their residual
estimate (Kahan/Parlett bound) of a closed-form eigenvalue, the largest nearest the
largest eigenvalue and not above it; the top Ritz vector mostly on the largest block."""
import numpy as np
import pytest

import synthgen as S

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

B, SZ = 51, 6554


@pytest.fixture(scope="module")
def blocks():
    n = B * SZ
    nnz = B * SZ * SZ
    rowptr = np.arange(n + 1, dtype=np.int64) * SZ
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    base = np.arange(SZ, dtype=np.int32)
    for b in range(B):
        z0 = b * SZ * SZ
        col[z0:z0 + SZ * SZ] = np.tile(base + b * SZ, SZ)
        val[z0:z0 + SZ * SZ] = (64 + b) / 128.0
    return S.CSR(n, rowptr, col, val)


def test_one_part_over_2g_nonzeros_closed_form(blocks):
    import paper_2201_07498_b200 as T
    A = blocks
    assert A.nnz > 2 ** 31
    lam = np.array([(64 + b) / 128.0 * SZ for b in range(B)])
    K, m = 8, 16
    with T.TopkEig(A, K, storage="f32", compute="f64", m=m, check_symmetry=False) as h:
        assert h.partition().tolist() == [0, A.n]
        x = np.random.default_rng(3).standard_normal(A.n)
        y = h.debug_spmv(x)
        r = h.solve(seed=1, vectors=True)
    # SpMV rows (f32 x, exact values): y_r = c_b * sum of the block's x, fp64 bound
    xr = x.astype(np.float32).astype(np.float64)
    bs = xr.reshape(B, SZ).sum(axis=1)
    babs = np.abs(xr).reshape(B, SZ).sum(axis=1)
    c = (64 + np.arange(B)) / 128.0
    yr = np.repeat(c * bs, SZ)
    bound = (SZ + 2) * 2.0 ** -53 * np.repeat(c * babs, SZ) + 2.0 ** -52 * np.abs(yr)
    assert np.all(np.abs(y - yr) <= bound)
    # Ritz values vs the closed form (Kahan/Parlett: each within its residual of some eigenvalue)
    assert r.info["k_found"] == K
    scale = lam.max()
    full = np.concatenate([lam, [0.0]])
    for th, est in zip(r.eigenvalues, r.residual_est):
        assert np.min(np.abs(full - th)) <= est * (1 + 1e-6) + 1e-9 * scale, (th, est)
    # m = 16 steps for 51 eigenvalues 0.9 % apart: the top pair is close, not converged;
    # Ritz values never exceed the spectrum, and the largest is nearest lambda_max
    assert r.eigenvalues[0] <= lam[-1] * (1 + 1e-12)
    assert abs(r.eigenvalues[0] - lam[-1]) < 0.5 * (lam[-1] - lam[-2])
    # the top Ritz vector has most of its weight on the largest block
    y0 = r.eigenvectors[0]
    w = np.linalg.norm(y0.reshape(B, SZ), axis=1)
    assert int(np.argmax(w)) == B - 1 and w[-1] >= 0.5
