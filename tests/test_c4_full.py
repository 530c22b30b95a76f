"""C4 at full size on one B200 (BASELINE.json configs[3]: R-MAT n = 1e8,
nnz ~ 1.5e9, FDF, K = m = 16).

test_c4_oracle_parity (default -m gpu run): the whole solve against a full
fp64 oracle solve (O3-O9, m = 16) on the same matrix and seed: all 16 Ritz
values normwise <= 1e-4, separated Ritz vectors <= 1e-5 (SURVEY 8(d) C4 row,
north-star gates), k_found / iterations / breakdown equal; then G = 8 loopback
parts (the 8-GPU partition on one device) against G = 1 (FDF
across G within 1e-6 normwise).

run_c4 (opt-in TOPK_C4=1 / TOPK_BIG=1 for C4X, > 2^31 nonzeros in one part):
sampled parity where the oracle can only afford single passes:
  * the SpMV kernel (Alg.1 l.9) on a seeded x, every row, against the oracle's
    fp64 SpMV with the rigorous per-row bound (len + 2) u sum |a x|;
  * alpha_1 = v1^T M v1 (Alg.1 l.10) against the oracle (same v1, reading Q8);
  * the top Ritz pair: true residual ||M y - theta y|| / |theta| (oracle SpMV
    on the GPU eigenvector) against the residual estimate |beta s_mk|.
Prints one "C4CHECK {json}" line per run (summarised under profiles/)."""
import json
import os
import time

import numpy as np
import pytest

import oracle as O
import synthgen as S

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def T():
    import paper_2201_07498_b200 as T
    return T


def run_c4(T, parts, name="C4"):
    out = {"config": name, "parts": parts}
    t0 = time.time()
    A = S.config_matrix(name)
    out.update(n=int(A.n), nnz=int(A.nnz), gen_s=round(time.time() - t0, 1))
    t0 = time.time()
    K, m = 16, 16
    with T.TopkEig(A, K, storage="f32", compute="f64", m=m, parts=parts, check_symmetry=False) as h:
        out["create_s"] = round(time.time() - t0, 1)
        out["_b"] = h.partition().tolist()
        # SpMV parity, every row
        x = np.random.default_rng(4).standard_normal(A.n)
        y = h.debug_spmv(x)
        xr = x.astype(np.float32).astype(np.float64)
        av = A.val.astype(np.float32).astype(np.float64)
        yr = O.spmv(A.rowptr, A.col, av, xr)
        absprod = O.spmv(A.rowptr, A.col, np.abs(av), np.abs(xr))
        bound = (np.diff(A.rowptr) + 2) * 2.0 ** -53 * absprod
        viol = int(np.sum(np.abs(y - yr) > bound))
        out["spmv_rows_checked"] = int(A.n)
        out["spmv_bound_violations"] = viol
        out["spmv_max_err_over_bound"] = float(np.max(np.abs(y - yr) / (bound + 1e-300)))
        del y, yr, absprod, bound
        # one solve, alpha_1 and the top Ritz pair
        t0 = time.time()
        r = h.solve(seed=1, vectors=True, vec_dtype="f32")
        out["solve_wall_s"] = round(time.time() - t0, 2)
        out["ms_solve_device"] = r.info["ms_solve"]
        alpha, beta, theta = h.tridiag()
    v1 = O.v1(1, A.n)
    v1 = v1 / np.linalg.norm(v1)
    a1 = float(np.dot(v1, O.spmv(A.rowptr, A.col, av, v1)))
    out["alpha1_gpu"] = float(alpha[0])
    out["alpha1_oracle"] = a1
    out["alpha1_rel_err"] = abs(alpha[0] - a1) / abs(a1)
    y0 = r.eigenvectors[0].astype(np.float64)
    th = float(r.eigenvalues[0])
    res = float(np.linalg.norm(O.spmv(A.rowptr, A.col, av, y0) - th * y0) / abs(th))
    out.update(theta1=th, residual_true_rel=res, residual_est_rel=float(r.residual_est[0] / abs(th)),
               k_found=int(r.info["k_found"]), iterations=int(r.info["iterations"]))
    b = np.asarray(out.pop("_b"))
    out["max_part_nnz"] = int(np.diff(A.rowptr[b]).max())
    print("C4CHECK " + json.dumps(out), flush=True)
    return out




@pytest.fixture(scope="module")
def c4():
    t0 = time.time()
    A = S.config_matrix("C4")
    print(f"C4 generated in {time.time() - t0:.1f} s: n={A.n} nnz={A.nnz}", flush=True)
    return A


def test_c4_oracle_parity(T, c4):
    from test_gpu_parity import check_solve, normwise
    A = c4
    K = m = 16
    out = {"config": "C4", "n": int(A.n), "nnz": int(A.nnz), "K": K, "m": m}
    t0 = time.time()
    with T.TopkEig(A, K, storage="f32", compute="f64", m=m) as h:  # symmetry check on
        out["create_s"] = round(time.time() - t0, 1)
        r1 = h.solve(seed=1, vectors=True, vec_dtype="f32")
        _, _, th1 = h.tridiag()
    t0 = time.time()
    ref = O.solve(A.rowptr, A.col, A.val, K=K, m=m, seed=1)
    out["oracle_s"] = round(time.time() - t0, 1)
    out["ritz_normwise_err"] = float(normwise(th1, ref.theta_all))
    assert out["ritz_normwise_err"] <= 1e-4
    check_solve(r1, ref, 1e-4)
    out["vec_max_err"] = float(max(min(np.linalg.norm(r1.eigenvectors[k] - ref.eigenvectors[k]),
                                       np.linalg.norm(r1.eigenvectors[k] + ref.eigenvectors[k]))
                                   for k in range(K)))
    del ref
    # the 8-GPU partition (rule P, 8 parts, padded replica) on one device vs one part
    with T.TopkEig(A, K, storage="f32", compute="f64", m=m, parts=8, check_symmetry=False) as h:
        r8 = h.solve(seed=1, vectors=False)
        _, _, th8 = h.tridiag()
    out["g8_vs_g1_normwise"] = float(normwise(th8, th1))
    assert out["g8_vs_g1_normwise"] <= 1e-6
    assert r8.info["iterations"] == r1.info["iterations"] and r8.info["k_found"] == K
    print("C4PARITY " + json.dumps(out), flush=True)


@pytest.mark.skipif(os.environ.get("TOPK_C4") != "1", reason="opt-in: TOPK_C4=1")
@pytest.mark.parametrize("parts", [1, 8])
def test_c4_full_size(T, parts):
    out = run_c4(T, parts)
    assert out["spmv_bound_violations"] == 0
    assert out["alpha1_rel_err"] <= 1e-6
    assert out["k_found"] == 16
    assert abs(out["residual_true_rel"] - out["residual_est_rel"]) <= 1e-4 + 1e-2 * out["residual_est_rel"]


@pytest.mark.skipif(os.environ.get("TOPK_BIG") != "1", reason="opt-in: TOPK_BIG=1 (~4 min, ~100 GB host RAM)")
def test_over_2g_nonzeros_one_part(T):
    """one part holding more than 2^31 nonzeros (64-bit
    physical offsets), n = 2^27 (GAP-kron's n), same sampled-parity checks."""
    out = run_c4(T, 1, "C4X")
    assert out["nnz"] > 2 ** 31 and out["max_part_nnz"] > 2 ** 31
    assert out["spmv_bound_violations"] == 0
    assert out["alpha1_rel_err"] <= 1e-6
    assert out["k_found"] == 16
    assert abs(out["residual_true_rel"] - out["residual_est_rel"]) <= 1e-4 + 1e-2 * out["residual_est_rel"]
