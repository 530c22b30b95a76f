"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs. Tolerances are BASELINE.json north_star's: Ritz values
within 1e-8 normwise in fp64 (DDD) and 1e-4 in mixed precision; eigenvector
residual <= 1e-5; partition and index layout bit-exact (DESIGN.md "Parity
contract"). Sizes span many SpMV tiles, long (split) rows and ragged tails."""
import numpy as np
import pytest

import oracle as O
import synthgen as S

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-8, "f32": 1e-4, "bf16": 1e-4}


@pytest.fixture(scope="module")
def T():
    import paper_2201_07498_b200 as T
    return T


@pytest.fixture(scope="module")
def c1():
    c = S.config_matrix("C1")
    rp, col, val = O.coo_to_csr(c.n, c.row, c.col, c.val)
    return c, S.CSR(c.n, rp, col, val)


@pytest.fixture(scope="module")
def c3s():
    return S.config_matrix("C3S")


def bf16_values(A):
    """A's values rounded to bf16 by the oracle's layout (O2), back in CSR order."""
    lrp, _, lv, _, perm = O.layout(A.rowptr, A.col, A.val, 1, np.array([0, A.n]), 0, "bf16", with_perm=True)
    idx = np.concatenate([np.arange(A.rowptr[r], A.rowptr[r + 1]) for r in perm]).astype(np.int64)
    out = np.empty_like(np.asarray(A.val, dtype=np.float64))
    out[idx] = lv
    return out


def normwise(a, b):
    a, b = np.sort(a), np.sort(b)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def check_solve(res, ref, tol, A=None, vec_tol=1e-5):
    th = ref.theta_all
    assert res.info["iterations"] == ref.lanczos.m_found
    assert bool(res.info["breakdown"]) == ref.lanczos.breakdown
    assert res.info["k_found"] == len(ref.eigenvalues)
    kf = len(ref.eigenvalues)
    err = np.abs(res.eigenvalues[:kf] - ref.eigenvalues).max() / abs(ref.eigenvalues[0])
    # selection can differ only where |theta_K| ~ |theta_K+1| within tol
    if err > tol:
        srt = np.sort(np.abs(th))[::-1]
        assert kf < len(th) and (srt[kf - 1] - srt[kf]) <= 2 * tol * abs(ref.eigenvalues[0]), err
    if res.eigenvectors is not None and ref.eigenvectors is not None:
        gaps = np.array([np.min(np.abs(np.delete(th, np.argmin(np.abs(th - t))) - t)) if len(th) > 1 else 1.0
                         for t in ref.eigenvalues]) / abs(ref.eigenvalues[0])
        for k in range(kf):
            y, yr = res.eigenvectors[k].astype(np.float64), ref.eigenvectors[k]
            assert abs(np.linalg.norm(y) - 1) < 1e-6
            if gaps[k] >= 1e-4 and abs(res.eigenvalues[k] - ref.eigenvalues[k]) <= tol * abs(ref.eigenvalues[0]):
                d = min(np.linalg.norm(y - yr), np.linalg.norm(y + yr))
                assert d <= vec_tol * max(1.0, 1e-4 / gaps[k]), (k, d, gaps[k])
                assert np.dot(y, yr) > 0, "sign convention <y, v1> > 0 differs"
    return err


# ------------------------------------------------------------------ layout
@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_layout_bit_exact_c1(T, c1, G, dtype):
    coo, csr = c1
    with T.TopkEig(coo, 8, storage=dtype if dtype != "bf16" else "f32", compute="f64",
                   values_storage=dtype, parts=G) as h:
        b = h.partition()
        assert np.array_equal(b, O.partition(csr.rowptr, G))
        for g in range(G):
            rp, col, val, npad = h.layout(g)
            orp, ocol, oval, onpad = O.layout(csr.rowptr, csr.col, csr.val, G, b, g, dtype)
            assert npad == onpad
            assert np.array_equal(rp, orp)
            assert np.array_equal(col, ocol)
            assert np.array_equal(val.view(np.uint64), oval.view(np.uint64))


@pytest.mark.parametrize("G,exchange", [(1, "allgather"), (4, "allgather"), (4, "halo")])
def test_layout_bit_exact_rmat(T, c3s, G, exchange):
    with T.TopkEig(c3s, 8, "f32", "f64", parts=G, exchange=exchange) as h:
        b = h.partition()
        assert np.array_equal(b, O.partition(c3s.rowptr, G))
        for g in range(G):
            rp, col, val, npad = h.layout(g)
            orp, ocol, oval, onpad = O.layout(c3s.rowptr, c3s.col, c3s.val, G, b, g, "f32")
            assert (npad, rp.tolist() == orp.tolist()) == (onpad, True)
            assert np.array_equal(col, ocol) and np.array_equal(val, oval)


# ------------------------------------------------------------------ SpMV
@pytest.mark.parametrize("name,storage,vals,G", [("C1", "f64", "f64", 1), ("C3S", "f64", "f64", 1),
                                                 ("C3S", "f32", "f32", 1), ("C3S", "f32", "bf16", 1),
                                                 ("C3S", "f64", "f64", 3)])
def test_spmv_parity(T, c1, c3s, name, storage, vals, G):
    A = c1[1] if name == "C1" else c3s
    x = np.random.default_rng(5).standard_normal(A.n)
    with T.TopkEig(A, 4, storage, "f64", values_storage=vals, parts=G) as h:
        y = h.debug_spmv(x)
    xr = x.astype(np.float32).astype(np.float64) if storage == "f32" else x
    if vals == "bf16":
        av = bf16_values(A)
    else:
        av = A.val if vals == "f64" else A.val.astype(np.float32).astype(np.float64)
    yr = O.spmv(A.rowptr, A.col, av, xr)
    absprod = O.spmv(A.rowptr, A.col, np.abs(av), np.abs(xr))
    rowlen = np.diff(A.rowptr)
    bound = (rowlen + 2) * 2.0 ** -53 * absprod
    assert np.all(np.abs(y - yr) <= bound + 1e-300), np.max(np.abs(y - yr) / (bound + 1e-300))


# ------------------------------------------------------------------ create: symmetry check on the device path
def test_create_rejects_asymmetric_on_device_host(T, c3s):
    """Row a2 through create on a GPU host: a one-entry value change, a dropped mirror
    entry and an asymmetric pattern are E_NOT_SYMMETRIC at G = 1 and 3, no handle is
    created, and the next create/solve in the same process is unaffected."""
    A = c3s
    r = int(np.argmax(np.diff(A.rowptr) > 3))
    k = A.rowptr[r] + 1
    val = A.val.copy(); val[k] += 2.0 ** -20
    drop_rp = A.rowptr.copy(); drop_rp[r + 1:] -= 1
    variants = [S.CSR(A.n, A.rowptr, A.col, val),
                S.CSR(A.n, drop_rp, np.delete(A.col, k), np.delete(A.val, k)),
                S.from_dense(np.array([[1.0, 2.0], [0.0, 1.0]]))]
    for V in variants:
        for G in (1, 3):
            with pytest.raises(T.TopkError) as e:
                T.TopkEig(V, 1, "f32", "f64", parts=min(G, V.n))
            assert e.value.status == 3
    ref = O.solve(A.rowptr, A.col, A.val, K=8, m=16, seed=2)
    res = T.solve(A, 8, storage="f64", compute="f64", m=16, seed=2)
    assert normwise(res.eigenvalues, ref.eigenvalues) <= 1e-8


# ------------------------------------------------------------------ small exact cases
def test_spec_examples(T, golden):
    for key in ("two_by_two", "antidiag_tie", "diag54321_top2"):
        ex = golden[key]
        A = S.from_dense(np.array(ex["A"], float) if "A" in ex else np.diag(ex["diag"]).astype(float))
        for st in ("f64", "f32"):
            r = T.solve(A, ex["K"], storage=st, compute="f64", m=ex.get("m", ex["K"]), seed=3)
            assert np.allclose(r.eigenvalues, ex["eigenvalues"], atol=1e-12 if st == "f64" else 1e-6), key
    ex = golden["identity4_breakdown"]
    r = T.solve(S.from_dense(np.eye(4)), 4, storage="f64", compute="f64", seed=5)
    assert r.info["breakdown"] == 1 and r.info["iterations"] == ex["m_found"]
    assert r.eigenvalues[0] == pytest.approx(1.0, abs=1e-15) and np.isnan(r.eigenvalues[1:]).all()
    ex = golden["alpha1_diag3210"]
    with T.TopkEig(S.from_dense(np.diag(ex["diag"]).astype(float)), 1, "f64", "f64") as h:
        h.solve(v1=np.array(ex["v1"]))
        a, b, t = h.tridiag()
        assert a[0] == ex["alpha1"]


@pytest.mark.parametrize("n", [12, 13, 40])
def test_cycle_breakdown(T, n):
    A = S.cycle_laplacian(n)
    ref = O.solve(A.rowptr, A.col, A.val, K=n, m=n, seed=4)
    r = T.solve(A, n, storage="f64", compute="f64", m=n, seed=4)
    assert r.info["breakdown"] == 1 and r.info["iterations"] == n // 2 + 1 == ref.lanczos.m_found
    assert normwise(r.eigenvalues[: r.info["k_found"]], ref.eigenvalues) <= 1e-12


def test_zero_and_tiny_matrices(T):
    Z = S.CSR(5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0))
    r = T.solve(Z, 2, storage="f64", compute="f64", check_symmetry=True)
    ref = O.solve(Z.rowptr, Z.col, Z.val, K=2, m=2, seed=1)
    assert r.info["iterations"] == ref.lanczos.m_found == 1 and r.info["breakdown"] == 1
    assert r.eigenvalues[0] == 0.0
    one = S.from_dense(np.array([[3.5]]))
    r = T.solve(one, 1, storage="f64", compute="f64")
    assert r.eigenvalues[0] == 3.5 and abs(abs(r.eigenvectors[0][0]) - 1) < 1e-15


# ------------------------------------------------------------------ full solves vs oracle
@pytest.mark.parametrize("m", [8, 64])
@pytest.mark.parametrize("storage,compute", [("f64", "f64"), ("f32", "f64")])
def test_c1_parity(T, c1, m, storage, compute):
    coo, csr = c1
    ref = O.solve(csr.rowptr, csr.col, csr.val, K=8, m=m, seed=1, tau=O.TAU[storage])
    r = T.solve(coo, 8, storage=storage, compute=compute, m=m, seed=1)
    assert normwise(T_all(T, coo, 8, storage, compute, m, 1), ref.theta_all) <= TOL[storage]
    check_solve(r, ref, TOL[storage])


def T_all(T, A, K, storage, compute, m, seed, **kw):
    with T.TopkEig(A, K, storage, compute, m=m, **kw) as h:
        h.solve(seed=seed, vectors=False)
        return h.tridiag()[2]


@pytest.mark.parametrize("K,m,storage,compute,vals", [
    (24, 24, "f32", "f64", None), (24, 96, "f32", "f64", None), (24, 24, "f64", "f64", None),
    (8, 64, "f64", "f64", None), (16, 48, "f32", "f32", None), (24, 24, "f32", "f64", "bf16")])
def test_rmat_parity(T, c3s, K, m, storage, compute, vals):
    A = c3s
    av = A.val
    if vals == "bf16":  # generator weights are bf16-exact: the matrix is unchanged
        assert np.array_equal(bf16_values(A), A.val)
    ref = O.solve(A.rowptr, A.col, av, K=K, m=m, seed=7, tau=O.TAU["f64"])
    r = T.solve(A, K, storage=storage, compute=compute, m=m, seed=7, values_storage=vals)
    th = T_all(T, A, K, storage, compute, m, 7, values_storage=vals)
    assert normwise(th, ref.theta_all) <= TOL[storage]
    check_solve(r, ref, TOL[storage])
    # converged pairs: true residual <= 1e-5 relative (north_star)
    conv = ref.residual_est <= 1e-7 * abs(ref.eigenvalues[0])
    import scipy.sparse as sp
    M = sp.csr_matrix((A.val, A.col, A.rowptr), shape=(A.n, A.n))
    for k in np.nonzero(conv)[0]:
        y = r.eigenvectors[k].astype(np.float64)
        assert np.linalg.norm(M @ y - r.eigenvalues[k] * y) <= 1e-5 * abs(ref.eigenvalues[0])


def test_basis_orthogonality(T, c3s):
    for storage, tol in (("f64", 1e-12), ("f32", 1e-5)):
        with T.TopkEig(c3s, 24, storage, "f64", m=48) as h:
            h.solve(seed=2, vectors=False)
            V = h.basis()
        assert np.abs(V @ V.T - np.eye(len(V))).max() <= tol


def test_cgs2_and_reorth_off(T, c3s):
    ref = O.solve(c3s.rowptr, c3s.col, c3s.val, K=16, m=32, seed=3)
    th2 = T_all(T, c3s, 16, "f64", "f64", 32, 3, reorth=2)
    assert normwise(th2, ref.theta_all) <= 1e-8
    # reorth off (paper's optional mode) is report-only: it runs,
    # and its basis is less orthogonal than with reorthogonalisation
    with T.TopkEig(c3s, 16, "f64", "f64", m=32, reorth=-1) as h:
        r = h.solve(seed=3)
        V = h.basis()
    with T.TopkEig(c3s, 16, "f64", "f64", m=32) as h:
        h.solve(seed=3)
        V1 = h.basis()
    assert np.isfinite(r.eigenvalues).all()
    assert np.abs(V @ V.T - np.eye(len(V))).max() > np.abs(V1 @ V1.T - np.eye(len(V1))).max()


@pytest.mark.parametrize("G,exchange", [(2, "allgather"), (3, "allgather"), (5, "allgather"),
                                        (2, "halo"), (5, "halo")])
def test_loopback_parts_match(T, c3s, G, exchange):
    """G row partitions (virtual ranks on one GPU): same answer as G = 1 within
    the cross-G tolerance (1e-12 DDD, 1e-6 FDF); layout per part. With
    the halo exchange (reading Q27) the SpMV reads the compact vectors."""
    for storage, tol in (("f64", 1e-12), ("f32", 1e-6)):
        th1 = T_all(T, c3s, 16, storage, "f64", 32, 5)
        thg = T_all(T, c3s, 16, storage, "f64", 32, 5, parts=G, exchange=exchange)
        assert normwise(thg, th1) <= tol
    ref = O.solve(c3s.rowptr, c3s.col, c3s.val, K=16, m=32, seed=5)
    r = T.solve(c3s, 16, storage="f64", compute="f64", m=32, seed=5, parts=G, exchange=exchange)
    check_solve(r, ref, 1e-8)


def test_halo_equals_allgather_bitwise(T, c3s):
    """The halo exchange moves exactly the values the SpMV reads, so the solve is
    bit-identical to the replicated-vector exchange (same kernels, same sums)."""
    out = []
    for ex in ("allgather", "halo"):
        with T.TopkEig(c3s, 8, "f32", "f64", m=24, parts=4, exchange=ex) as h:
            out.append(h.solve(seed=12))
            y = h.debug_spmv(np.linspace(-1, 1, c3s.n))
            out.append(y)
    assert np.array_equal(out[0].eigenvalues, out[2].eigenvalues)
    assert np.array_equal(out[0].eigenvectors, out[2].eigenvectors)
    assert np.array_equal(out[1], out[3])


def test_determinism(T, c3s):
    with T.TopkEig(c3s, 24, "f32", "f64", m=48) as h:
        a = h.solve(seed=11)
        b = h.solve(seed=11)
        c = h.solve(seed=12)
    assert np.array_equal(a.eigenvalues, b.eigenvalues)
    assert np.array_equal(a.eigenvectors, b.eigenvectors)
    assert not np.array_equal(a.eigenvalues, c.eigenvalues)


def test_eager_equals_graph(T, c3s):
    with T.TopkEig(c3s, 8, "f32", "f64", m=16, use_graph=False) as h:
        a = h.solve(seed=4)
    with T.TopkEig(c3s, 8, "f32", "f64", m=16) as h:
        b = h.solve(seed=4)
    assert np.array_equal(a.eigenvalues, b.eigenvalues)
    assert np.array_equal(a.eigenvectors, b.eigenvectors)


def test_async_api(T, c3s):
    import torch
    with T.TopkEig(c3s, 8, "f32", "f64", m=16) as h:
        r = h.solve(seed=9, vec_dtype="f32")
        ev = torch.zeros(8, dtype=torch.float64, device="cuda")
        Y = torch.zeros(8, c3s.n, dtype=torch.float32, device="cuda")
        h.solve_async(9, ev.data_ptr(), Y.data_ptr(), "f32")
        info = h.sync()
    assert info["k_found"] == 8
    assert np.array_equal(ev.cpu().numpy(), r.eigenvalues)
    assert np.array_equal(Y.cpu().numpy(), r.eigenvectors)


# ------------------------------------------------------------------ closed forms at C2 size
@pytest.mark.parametrize("storage,tol", [("f64", 1e-13), ("f32", 1e-8)])
def test_dirichlet_1M_closed_form(T, storage, tol):
    n = 1_000_000
    A = S.dirichlet(n)
    j = np.arange(1, n + 1)
    ks = 58_823 * np.arange(1, 17)
    v1 = np.zeros(n)
    for k in ks:
        v1 += np.sin(np.pi * k * j / (n + 1))
    r = T.solve(A, 16, storage=storage, compute="f64", m=16, v1=v1, vectors=False,
                breakdown_tol=1e-300)
    lam = 2 - 2 * np.cos(np.pi * ks / (n + 1))
    assert np.abs(np.sort(r.eigenvalues) - np.sort(lam)).max() <= tol


# ------------------------------------------------------------------ full C3 size
def test_c3_full_size_parity(T):
    """BASELINE config C3 at full size (R-MAT n = 4,194,304, nnz ~ 61M), FDF,
    K = m = 24, in the launch configuration bench.py times: vs the oracle."""
    A = S.config_matrix("C3")
    ref = O.solve(A.rowptr, A.col, A.val, K=24, m=24, seed=1)
    r = T.solve(A, 24, storage="f32", compute="f64", m=24, seed=1, vec_dtype="f32", check_symmetry=False)
    check_solve(r, ref, 1e-4)


# ------------------------------------------------------------------ v1 bit-exact (SURVEY 8(c) parity contract)
@pytest.mark.parametrize("storage,G", [("f64", 1), ("f32", 1), ("f64", 3), ("bf16", 1)])
def test_v1_unnormalised_bit_exact(T, c3s, storage, G):
    """The unnormalised start vector u_r = 2 U(h3(seed, 0x7631, r)) - 1 (reading Q8,
    PAPER.md:75,205) stored as basis column 0 equals the oracle's orc_v1 bit for bit
    after the one storage rounding (f64: identical; f32 / bf16: RNE straight from f64,
    reading Q22), over every global row, for every part."""
    seed = 12345
    n = c3s.n
    u = O.v1(seed, n)
    # the oracle's storage rounding (O2 layout rule) of a diagonal matrix holding u:
    # every row has degree 1, so the degree order is the original order
    rp = np.arange(n + 1, dtype=np.int64)
    _, _, want, _ = O.layout(rp, np.arange(n, dtype=np.int32), u, 1, np.array([0, n]), 0, storage)
    with T.TopkEig(c3s, 8, storage, "f64", m=8, parts=G) as h:
        h.solve(seed=seed, vectors=False)
        b = h.partition()
        got = np.empty(n)
        for g in range(G):
            got[b[g]:b[g + 1]] = h.basis(g, raw=True)[0]
    assert np.array_equal(np.asarray(want, np.float64).view(np.uint64), got.view(np.uint64))


# ------------------------------------------------------------------ closed form, random start (P5 via the ABI)
@pytest.mark.parametrize("kind", ["dirichlet", "cycle"])
def test_kahan_bound_1M_random_start(T, kind):
    """C2 (n = 1e6), random v1, K = m = 16: every Ritz value lies within its true
    residual ||A y - theta y|| of a closed-form eigenvalue (Kahan/Parlett bound;
    SURVEY P5), residual computed by the oracle's SpMV on the GPU eigenvector."""
    n = 1_000_000
    A = S.dirichlet(n) if kind == "dirichlet" else S.cycle_laplacian(n)
    r = T.solve(A, 16, storage="f64", compute="f64", m=16, seed=3)
    k = np.arange(1, n + 1) if kind == "dirichlet" else np.arange(n)
    lam = np.sort(2 - 2 * np.cos((np.pi if kind == "dirichlet" else 2 * np.pi) * k / ((n + 1) if kind == "dirichlet" else n)))
    for th, y in zip(r.eigenvalues, r.eigenvectors):
        res = np.linalg.norm(O.spmv(A.rowptr, A.col, A.val, y) - th * y)
        i = np.searchsorted(lam, th)
        gap = min(abs(lam[min(i, n - 1)] - th), abs(lam[max(i - 1, 0)] - th))
        assert gap <= res * (1 + 1e-6) + 1e-12


# ------------------------------------------------------------------ full C3 size, fp64
def test_c3_full_size_parity_ddd(T):
    """C3 at full size in DDD (f64 storage and compute): Ritz values within
    1e-8 normwise of the oracle, vectors within 1e-5 (north-star gates)."""
    A = S.config_matrix("C3")
    ref = O.solve(A.rowptr, A.col, A.val, K=24, m=24, seed=2)
    r = T.solve(A, 24, storage="f64", compute="f64", m=24, seed=2, check_symmetry=False)
    check_solve(r, ref, 1e-8)


@pytest.mark.parametrize("m", [64, 130, 192, 300])
@pytest.mark.parametrize("cluster", [True, False])
def test_large_m_jacobi_paths(T, c3s, m, cluster):
    """Krylov dimensions whose T, S do not fit one SM's shared memory: the
    cluster-distributed Jacobi (8 CTAs at m = 64; 16 at m = 130, 192, 300) and the
    single-CTA global-memory fallback both match the oracle (reading Q10)."""
    ref = O.solve(c3s.rowptr, c3s.col, c3s.val, K=24, m=m, seed=8)
    with T.TopkEig(c3s, 24, "f64", "f64", m=m, jacobi_path="auto" if cluster else "single") as h:
        r = h.solve(seed=8)
        _, _, th = h.tridiag()
    assert r.info["jacobi_converged"] == 1
    assert normwise(th, ref.theta_all) <= 1e-8
    check_solve(r, ref, 1e-8)


def test_memory_pool_reuse_and_trim(T, c3s):
    """Handles created after a destroy reuse the cached device blocks (same
    results), and topk_eig_trim_pool releases them."""
    with T.TopkEig(c3s, 8, "f32", "f64", m=16) as h:
        a = h.solve(seed=2)
    with T.TopkEig(c3s, 8, "f32", "f64", m=16) as h:
        b = h.solve(seed=2)
    assert np.array_equal(a.eigenvalues, b.eigenvalues) and np.array_equal(a.eigenvectors, b.eigenvectors)
    assert T.trim_pool() > 0
    assert T.trim_pool() == 0


@pytest.mark.parametrize("storage,tol", [("f64", 1e-8), ("f32", 1e-4)])
def test_periodic_reorth(T, c3s, storage, tol):
    """Reading Q28: reorthogonalisation of the pairs of iterations (4k, 4k + 1) only,
    against oracle.solve_periodic, within the north-star tolerances; period 1 is the
    default path bit for bit."""
    K, m, p = 16, 32, 4
    ref = O.solve_periodic(c3s.rowptr, c3s.col, c3s.val, K, m, p, seed=6, tau=O.TAU[storage])
    th = T_all(T, c3s, K, storage, "f64", m, 6, reorth_period=p)
    assert normwise(th, ref.theta_all) <= tol
    a = T_all(T, c3s, K, storage, "f64", m, 6, reorth_period=1)
    b = T_all(T, c3s, K, storage, "f64", m, 6)
    assert np.array_equal(a, b)


def test_bf16_vectors_report_only(T, c3s):
    """bf16 vector storage (reading Q21: report-only, unstable as the paper says):
    the bf16 kernels run end to end; the dominant, well separated eigenvalue is
    still found to bf16 accuracy and the returned vectors are unit norm."""
    ref = O.solve(c3s.rowptr, c3s.col, c3s.val, K=8, m=16, seed=2)
    with T.TopkEig(c3s, 8, "bf16", "f64", values_storage="bf16", m=16) as h:
        r = h.solve(seed=2, vectors=True, vec_dtype="f32")
    assert r.info["k_found"] == 8 and np.all(np.isfinite(r.eigenvalues))
    assert abs(r.eigenvalues[0] - ref.eigenvalues[0]) <= 1e-2 * abs(ref.eigenvalues[0])
    assert np.allclose(np.linalg.norm(r.eigenvectors.astype(np.float64), axis=1), 1.0, atol=1e-3)


@pytest.mark.parametrize("G", [1, 3])
def test_row_length_boundaries(T, G):
    """Rows of degree exactly at the layout boundaries -- 127/128 (SELL) vs 129 (big
    row), 8191/8192 (one chunk) vs 8193 and 16385 (several chunks, finished by the last
    arriving one) -- plus empty rows and a ragged tail: every SpMV row within the
    rigorous fp64 bound of the oracle, and the solve at the DDD tolerance."""
    A = S.stars([8191, 8192, 8193, 16385], dense=[127, 128, 129, 3])
    x = np.random.default_rng(1).standard_normal(A.n)
    with T.TopkEig(A, 8, "f64", "f64", m=24, parts=G) as h:
        y = h.debug_spmv(x)
        r = h.solve(seed=2)
    yr = O.spmv(A.rowptr, A.col, A.val, x)
    bound = (np.diff(A.rowptr) + 2) * 2.0 ** -53 * O.spmv(A.rowptr, A.col, np.abs(A.val), np.abs(x))
    assert np.all(np.abs(y - yr) <= bound)
    ref = O.solve(A.rowptr, A.col, A.val, K=8, m=24, seed=2)
    check_solve(r, ref, 1e-8)


@pytest.mark.parametrize("storage,tol", [("f64", 1e-8), ("f32", 1e-4)])
def test_partial_reorth(T, c3s, storage, tol):
    """Reading Q29: partial reorthogonalisation (reorth = 3) against oracle.solve_pro:
    the same number of reorthogonalisation passes (the decisions come from Simon's
    estimate in the same arithmetic order), Ritz values within the north-star
    tolerances, and (fp64) far fewer passes than iterations."""
    K, m, seed = 16, 64, 6
    eps = 2.0 ** -53 if storage == "f64" else 2.0 ** -24
    ref = O.solve_pro(c3s.rowptr, c3s.col, c3s.val, K, m, eps, seed=seed, tau=O.TAU[storage])
    with T.TopkEig(c3s, K, storage, "f64", m=m, reorth=3) as h:
        r = h.solve(seed=seed, vectors=False)
        th = h.tridiag()[2]
    assert r.info["reorth_passes"] == len(ref.extra["reorth_steps"]), (r.info["reorth_passes"], ref.extra["reorth_steps"])
    # fp64 vectors: a fraction of the iterations; f32 vectors (eps = 2^-24) reach the
    # sqrt(eps) level within a few steps, so most iterations take the pass
    assert 0 < r.info["reorth_passes"] < (m // 2 if storage == "f64" else m)
    assert normwise(th, ref.theta_all) <= tol


# ------------------------------------------------------------------ info: phase times
def test_info_phase_times(T, c3s):
    """topk_eig_info_t ms_lanczos + ms_jacobi + ms_ritz partition ms_solve (events at the
    phase boundaries inside the graph); one process: no interconnect bytes."""
    with T.TopkEig(c3s, 8, "f32", "f64", m=24) as h:
        for _ in range(2):
            r = h.solve(seed=3)
    i = r.info
    assert i["ms_lanczos"] > 0 and i["ms_jacobi"] > 0 and i["ms_ritz"] > 0
    assert abs(i["ms_lanczos"] + i["ms_jacobi"] + i["ms_ritz"] - i["ms_solve"]) <= 0.02 * i["ms_solve"] + 0.01
    assert i["bytes_nvlink"] == 0


# ------------------------------------------------------------------ two-pass SpMV (overlapped exchange)
@pytest.mark.parametrize("G", [2, 3, 8])
def test_two_pass_spmv_overlap(T, c3s, G):
    """The SpMV as two passes, own-slot columns first (what one
    process per GPU runs so the vector allgather overlaps the first pass), on G loopback
    parts (overlap = 1: the same kernels and sums as the multi-process run): every SpMV row
    within the rigorous fp64 bound, the layout export (both passes merged back into
    canonical order) bit-exact against the oracle, the DDD solve within 1e-12 of the one-pass
    solve and within the parity tolerance of the oracle, bitwise repeatable."""
    x = np.random.default_rng(13).standard_normal(c3s.n)
    with T.TopkEig(c3s, 8, "f64", "f64", m=24, parts=G, overlap=1) as h:
        y = h.debug_spmv(x)
        r = h.solve(seed=5)
        r2 = h.solve(seed=5)
        b = h.partition()
        for g in range(G):
            rp, col, val, npad = h.layout(g)
            orp, ocol, oval, onpad = O.layout(c3s.rowptr, c3s.col, c3s.val, G, b, g, "f64")
            assert npad == onpad and np.array_equal(rp, orp)
            assert np.array_equal(col, ocol) and np.array_equal(val.view(np.uint64), oval.view(np.uint64))
    yr = O.spmv(c3s.rowptr, c3s.col, c3s.val, x)
    bound = (np.diff(c3s.rowptr) + 2) * 2.0 ** -53 * O.spmv(c3s.rowptr, c3s.col, np.abs(c3s.val), np.abs(x))
    assert np.all(np.abs(y - yr) <= bound + 1e-300)
    assert np.array_equal(r.eigenvalues, r2.eigenvalues) and np.array_equal(r.eigenvectors, r2.eigenvectors)
    with T.TopkEig(c3s, 8, "f64", "f64", m=24, parts=G, overlap=-1) as h:
        r0 = h.solve(seed=5)
    assert np.abs(r.eigenvalues - r0.eigenvalues).max() <= 1e-12 * abs(r0.eigenvalues[0])
    ref = O.solve(c3s.rowptr, c3s.col, c3s.val, K=8, m=24, seed=5)
    check_solve(r, ref, 1e-8)


def test_two_pass_spmv_fdf_row_boundaries(T):
    """Two-pass SpMV on rows at the chunk / SELL boundaries (stars), FDF, G = 3 loopback:
    rows whose entries are all own-slot or all remote, empty rows, ragged tail."""
    A = S.stars([8191, 8192, 8193, 16385], dense=[127, 128, 129, 3])
    x = np.random.default_rng(2).standard_normal(A.n)
    with T.TopkEig(A, 8, "f32", "f64", m=24, parts=3, overlap=1) as h:
        y = h.debug_spmv(x)
        r = h.solve(seed=2)
    xr = x.astype(np.float32).astype(np.float64)
    av = A.val.astype(np.float32).astype(np.float64)
    yr = O.spmv(A.rowptr, A.col, av, xr)
    bound = (np.diff(A.rowptr) + 2) * 2.0 ** -53 * O.spmv(A.rowptr, A.col, np.abs(av), np.abs(xr))
    assert np.all(np.abs(y - yr) <= bound + 1e-300)
    ref = O.solve(A.rowptr, A.col, A.val, K=8, m=24, seed=2)
    check_solve(r, ref, 1e-4)


# ------------------------------------------------------------------ Ritz output on the fp64 tensor cores
@pytest.mark.parametrize("K,m,storage", [(5, 12, "f64"), (16, 40, "f32"), (40, 64, "f64"), (40, 64, "f32")])
def test_ritz_mma_paths(T, c3s, K, m, storage):
    """k_ritz_mma (mma.sync m8n8k4 f64; 1, 2 or 4 output tiles per warp, several output
    groups at K = 40) against the CUDA-core k_ritz and the oracle: vectors within 1e-12
    (f64) / 1e-6 (f32 outputs) of the CUDA-core path, parity with the oracle."""
    out = {}
    for path in ("auto", "cuda_cores"):
        with T.TopkEig(c3s, K, storage, "f64", m=m, ritz_path=path) as h:
            out[path] = h.solve(seed=6, vectors=True, vec_dtype="f64")
    a, b = out["auto"], out["cuda_cores"]
    assert np.array_equal(a.eigenvalues, b.eigenvalues)
    tol = 1e-12 if storage == "f64" else 1e-6
    for k in range(len(a.eigenvalues)):
        assert np.linalg.norm(a.eigenvectors[k] - b.eigenvectors[k]) <= tol
    ref = O.solve(c3s.rowptr, c3s.col, c3s.val, K=K, m=m, seed=6)
    # FDF at K = 40: the deeper Ritz pairs have relative gaps ~2e-4, where f32 storage
    # moves a vector by ~1e-5 (the error of the pair / its gap); the paths agree exactly above
    check_solve(a, ref, 1e-8 if storage == "f64" else 1e-4, vec_tol=1e-5 if storage == "f64" or K <= 24 else 5e-5)
