"""Pins of the CPU oracle (oracle/) against things other than itself.

Each test names the pin of DESIGN.md "Oracle pins" (P1..P10) it implements and
the oracle step(s) it covers. These run on CPU (-m "not gpu").
"""
import itertools
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle as O
import synthgen as S


def csr_of(a):
    m = S.from_dense(a)
    return m.rowptr, m.col, m.val


def er_csr(n, samples, seed):
    c = S.er_coo(n, samples, seed)
    return O.coo_to_csr(n, c.row, c.col, c.val)


def dense(n, rp, c, v):
    return sp.csr_matrix((v, c, rp), shape=(n, n)).toarray()


# ---------------------------------------------------------------- P10 (O1)
def test_p10_coo_spec_examples(golden):
    for ex in golden["coo"]:
        e = np.array(ex["entries"], dtype=float).reshape(-1, 3)
        rp, c, v = O.coo_to_csr(ex["n"], e[:, 0].astype(np.int64), e[:, 1].astype(np.int32),
                                e[:, 2])
        assert rp.tolist() == ex["rowptr"], ex["cite"]
        assert c.tolist() == ex["col"], ex["cite"]
        assert v.tolist() == ex["val"], ex["cite"]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_p10_coo_duplicates_vs_dense_accumulation(seed):
    """Duplicate summation == dense accumulation; round trip CSR->COO->CSR is the identity."""
    rng = np.random.default_rng(seed)
    n, nnz = 40, 600
    r = rng.integers(0, n, nnz)
    c = rng.integers(0, n, nnz).astype(np.int32)
    v = rng.integers(-8, 9, nnz).astype(float) / 4  # exact sums in any order
    rp, cc, vv = O.coo_to_csr(n, r, c, v)
    d = np.zeros((n, n))
    np.add.at(d, (r, c), v)
    occupied = np.zeros((n, n), bool)
    occupied[r, c] = True
    assert np.array_equal(dense(n, rp, cc, vv), d)
    assert len(vv) == occupied.sum()
    for row in range(n):  # sorted, unique columns
        cols = cc[rp[row]:rp[row + 1]]
        assert np.all(np.diff(cols) > 0)
    rows = np.repeat(np.arange(n), np.diff(rp))
    rp2, c2, v2 = O.coo_to_csr(n, rows, cc, vv)
    assert np.array_equal(rp2, rp) and np.array_equal(c2, cc) and np.array_equal(v2, vv)


def test_p10_coo_rejects_out_of_range():
    with pytest.raises(ValueError):
        O.coo_to_csr(3, np.array([0, 3]), np.array([0, 0], np.int32), np.ones(2))
    with pytest.raises(ValueError):
        O.coo_to_csr(3, np.array([0, 1]), np.array([0, -1], np.int32), np.ones(2))


def test_p10_symmetry_check():
    rp, c, v = er_csr(200, 1000, 5)
    assert O.is_symmetric(200, rp, c, v)
    d = dense(200, rp, c, v)
    assert np.array_equal(d, d.T)
    v2 = v.copy()
    k = np.nonzero(c != np.repeat(np.arange(200), np.diff(rp)))[0][0]
    v2[k] = np.nextafter(v2[k], 10)  # one-ulp asymmetry
    assert not O.is_symmetric(200, rp, c, v2)
    # structural asymmetry: drop one off-diagonal entry
    rows = np.repeat(np.arange(200), np.diff(rp))
    keep = np.ones(len(v), bool)
    keep[k] = False
    rp3, c3, v3 = O.coo_to_csr(200, rows[keep], c[keep], v[keep])
    assert not O.is_symmetric(200, rp3, c3, v3)


# ---------------------------------------------------------------- P9 (O2)
def brute_partition(rownnz, G):
    n = len(rownnz)
    pre = np.concatenate([[0], np.cumsum(rownnz)])
    best = None
    for cuts in itertools.combinations(range(1, n), G - 1):
        b = (0,) + cuts + (n,)
        load = max(pre[b[k + 1]] - pre[b[k]] for k in range(G))
        key = (load, b)
        if best is None or key < best:
            best = key
    return list(best[1])


def test_p9_partition_spec_examples(golden):
    for ex in golden["partition"]:
        rp = np.concatenate([[0], np.cumsum(ex["row_nnz"])]).astype(np.int64)
        assert O.partition(rp, ex["G"]).tolist() == ex["boundaries"], ex["cite"]


def test_p9_partition_equals_brute_force():
    rng = np.random.default_rng(7)
    cases = 0
    for _ in range(3000):
        n = int(rng.integers(1, 10))
        G = int(rng.integers(1, n + 1))
        rownnz = rng.integers(0, 6, n) * (rng.random(n) > 0.3)
        rp = np.concatenate([[0], np.cumsum(rownnz)]).astype(np.int64)
        assert O.partition(rp, G).tolist() == brute_partition(rownnz, G), (rownnz, G)
        cases += 1
    assert cases == 3000


def test_p9_partition_invalid():
    with pytest.raises(ValueError):
        O.partition(np.array([0, 1, 2]), 3)


# ---------------------------------------------------------------- layout (O2)
@pytest.mark.parametrize("G", [1, 2, 3, 5])
@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_layout_reassembles_matrix(G, dtype):
    """Concatenated partitions, rows and columns mapped back through the
    hub-first positions, give back M (values rounded)."""
    rp, c, v = er_csr(500, 3000, 11)
    b = O.partition(rp, G)
    npad_expect = int(math.ceil(max(np.diff(b)) / 64) * 64)
    parts = [O.layout(rp, c, v, G, b, g, dtype, with_perm=True) for g in range(G)]
    perms = [pt[4] for pt in parts]
    dense = np.zeros((500, 500))
    np.add.at(dense, (np.repeat(np.arange(500), np.diff(rp)), c), v)
    got = np.zeros((500, 500))
    for g, (lrp, lc, lv, npad, perm) in enumerate(parts):
        assert npad == npad_expect
        assert lrp[0] == 0 and len(lrp) == b[g + 1] - b[g] + 1
        assert sorted(perm) == list(range(b[g + 1] - b[g]))
        owner, local = lc // npad, lc % npad
        assert np.all(local < np.diff(b)[owner])
        gcol = np.array([b[o] + perms[o][q] for o, q in zip(owner, local)], np.int64)
        grow = b[g] + np.repeat(perm, np.diff(lrp))
        np.add.at(got, (grow, gcol), lv)
    if dtype == "f64":
        assert np.array_equal(got, dense)
    elif dtype == "f32":
        assert np.array_equal(got, dense.astype(np.float32).astype(np.float64))
    else:
        nz = dense != 0
        check_bf16_rounding(dense[nz], got[nz])


def test_degree_order_positions_brute_force():
    """Inside each part: rows by (degree desc, index asc), so empty rows last
    (DESIGN.md 2)."""
    rp, c, v = er_csr(300, 200, 3)
    deg = np.diff(rp)
    assert (deg == 0).any()
    for G in (1, 2, 3):
        b = O.partition(rp, G)
        pos = O.positions(rp, G, b)
        for g in range(G):
            rows = list(range(b[g], b[g + 1]))
            order = sorted(rows, key=lambda r: (-deg[r], r))
            assert [pos[r] for r in order] == list(range(len(rows)))


def check_bf16_rounding(x, r):
    """r is x rounded to 8 significant bits, to nearest, ties to even (property pin)."""
    nz = x != 0
    e = np.floor(np.log2(np.abs(x[nz])))
    ulp = 2.0 ** (e - 7)
    q = r[nz] / ulp
    assert np.all(q == np.round(q)), "not on the bf16 grid"
    assert np.all(np.abs(r[nz] - x[nz]) <= ulp / 2 * (1 + 1e-15) + 2.0 ** (e - 8) * 0), "not nearest"
    tie = np.abs(np.abs(r[nz] - x[nz]) - ulp / 2) == 0
    assert np.all((q[tie] % 2) == 0), "tie not to even"


def test_bf16_rounding_ties():
    """Exact midpoints between bf16 neighbours round to the even mantissa."""
    x = np.array([1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 1 + 2 ** -8 + 2 ** -30, 0.75])
    rp = np.arange(len(x) + 1, dtype=np.int64)
    c = np.arange(len(x), dtype=np.int32)
    _, _, lv, _ = O.layout(rp, c, x, 1, np.array([0, len(x)]), 0, "bf16")
    assert lv.tolist() == [1.0, 1 + 4 * 2 ** -8, -1.0, 1 + 2 * 2 ** -8, 0.75]


# ---------------------------------------------------------------- O3 v1
def splitmix_first(state):
    m = (1 << 64) - 1
    z = (state + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def test_v1_hash_pinned_to_splitmix64_vector(golden):
    # the Python mix below is anchored by the published splitmix64 test vector ...
    assert splitmix_first(0) == int(golden["splitmix64"]["state0_first_output"], 16)

    def h3(s, a, b):
        return splitmix_first(splitmix_first(splitmix_first(s) ^ a) ^ b)

    # ... and the oracle's v1 entries equal it bit for bit (reading Q8)
    for seed in (0, 1, 12345):
        u = O.v1(seed, 50)
        ref = [2.0 * ((h3(seed, 0x7631, r) >> 11) * 2.0 ** -53) - 1.0 for r in range(50)]
        assert u.tolist() == ref
    u = O.v1(3, 100000)
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.01


# ---------------------------------------------------------------- SpMV (l.9)
def test_spmv_vs_scipy():
    rp, c, v = er_csr(700, 5000, 2)
    x = np.random.default_rng(0).standard_normal(700)
    y = O.spmv(rp, c, v, x)
    yr = sp.csr_matrix((v, c, rp), shape=(700, 700)) @ x
    assert np.allclose(y, yr, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- P2 (O7)
def test_p2_jacobi_spec_examples():
    th, Sm, sw, conv = O.jacobi(np.array([[2.0, 1], [1, 2]]))
    assert conv
    order = np.argsort(-th)
    assert np.allclose(th[order], [3, 1], atol=1e-15)
    v3 = Sm[:, order[0]] * np.sign(Sm[0, order[0]])
    v1 = Sm[:, order[1]] * np.sign(Sm[0, order[1]])
    assert np.allclose(v3, [2 ** -0.5, 2 ** -0.5], atol=1e-15)
    assert np.allclose(v1, [2 ** -0.5, -2 ** -0.5], atol=1e-15)
    th, Sm, sw, conv = O.jacobi(np.eye(6))
    assert conv and sw == 1 and np.array_equal(Sm, np.eye(6)) and np.array_equal(th, np.ones(6))


@pytest.mark.parametrize("m", [2, 3, 8, 24, 64])
def test_p2_jacobi_vs_eigh_and_invariants(m):
    rng = np.random.default_rng(m)
    for trial in range(3):
        if trial == 0:  # random tridiagonal (the shape Lanczos produces)
            A = np.diag(rng.standard_normal(m))
            off = rng.random(m - 1) + 0.01
            A += np.diag(off, 1) + np.diag(off, -1)
        else:
            B = rng.standard_normal((m, m))
            A = (B + B.T) / 2
        th, Sm, sw, conv = O.jacobi(A)
        assert conv
        ref = np.linalg.eigvalsh(A)
        nrm = np.linalg.norm(A, 2)
        assert np.allclose(np.sort(th), ref, rtol=0, atol=1e-13 * nrm)
        assert abs(th.sum() - np.trace(A)) <= 1e-13 * nrm * m
        assert np.abs(Sm.T @ Sm - np.eye(m)).max() <= 1e-13 * m
        assert np.abs(A @ Sm - Sm * th).max() <= 1e-13 * nrm * m


def test_p2_jacobi_sweep_cap():
    rng = np.random.default_rng(1)
    B = rng.standard_normal((20, 20))
    th, Sm, sw, conv = O.jacobi(B + B.T, max_sweeps=1)
    assert sw == 1 and not conv


# ---------------------------------------------------------------- P3 (O4-O8)
def test_p3_alpha1(golden):
    ex = golden["alpha1_diag3210"]
    rp, c, v = csr_of(np.diag(ex["diag"]).astype(float))
    lz = O.lanczos(rp, c, v, np.array(ex["v1"]), 1)
    assert lz.alpha[0] == ex["alpha1"], ex["cite"]


def test_p3_identity_breakdown(golden):
    ex = golden["identity4_breakdown"]
    rp, c, v = csr_of(np.eye(ex["n"]))
    r = O.solve(rp, c, v, K=4, m=4, seed=5)
    assert r.lanczos.breakdown and r.lanczos.m_found == ex["m_found"], ex["cite"]
    assert np.allclose(r.eigenvalues, [ex["eigenvalue"]], atol=1e-15)


@pytest.mark.parametrize("key", ["two_by_two", "antidiag_tie", "diag54321_top2"])
def test_p3_small_solves(golden, key):
    ex = golden[key]
    A = np.array(ex["A"], float) if "A" in ex else np.diag(ex["diag"]).astype(float)
    rp, c, v = csr_of(A)
    r = O.solve(rp, c, v, K=ex["K"], m=ex.get("m", ex["K"]), seed=3)
    assert np.allclose(r.eigenvalues, ex["eigenvalues"], rtol=0, atol=1e-14), ex["cite"]


def test_p3_orthogonalisation_example(golden):
    """basis {e1}, v = e1 + e2 -> e2. Lanczos on diag(1,0,0) from
    v1 = e1 makes v_nxt = M e1 - alpha_1 e1 = 0 -> breakdown; use the MGS step on
    A = [[0,1,0],[1,0,0],[0,0,0]] with v1 = e1: y = e2, alpha_1 = 0, w = e2."""
    A = np.array([[0.0, 1, 0], [1, 0, 0], [0, 0, 0]])
    rp, c, v = csr_of(A)
    lz = O.lanczos(rp, c, v, np.array([1.0, 0, 0]), 2)
    assert lz.V[1].tolist() == golden["orth_e1"]["result"]


# ---------------------------------------------------------------- P1 (O3-O7)
@pytest.mark.parametrize("n,samples,seed", [(40, 100, 1), (120, 500, 2), (300, 900, 3)])
def test_p1_full_dimension_lanczos_equals_eigh(n, samples, seed):
    rp, c, v = er_csr(n, samples, seed)
    A = dense(n, rp, c, v)
    r = O.solve(rp, c, v, K=n, m=n, seed=seed)
    ref = np.linalg.eigvalsh(A)
    nrm = np.linalg.norm(A, 2)
    mf = r.lanczos.m_found
    if mf == n:
        assert np.allclose(np.sort(r.theta_all), ref, rtol=0, atol=1e-10 * nrm)
    else:  # invariant subspace hit: every Ritz value is an eigenvalue
        d = np.abs(r.theta_all[:, None] - ref[None, :]).min(axis=1)
        assert d.max() <= 1e-10 * nrm


# ---------------------------------------------------------------- P4 (O3-O9)
def test_p4_dirichlet_1M_closed_form():
    """Dirichlet tridiag(-1,2,-1), n = 10^6, K = m = 16, v1 = sum of 16 spread sine
    modes k_i = 58,823 i: the Krylov space is exactly their span, so the Ritz
    values are the closed-form eigenvalues 2 - 2cos(pi k_i/(n+1))."""
    n = 1_000_000
    A = S.dirichlet(n)
    j = np.arange(1, n + 1)
    ks = 58_823 * np.arange(1, 17)
    v1 = np.zeros(n)
    for k in ks:
        v1 += np.sin(np.pi * k * j / (n + 1))
    r = O.solve(A.rowptr, A.col, A.val, K=16, m=16, v1vec=v1, tau=0.0, want_vectors=False)
    lam = 2 - 2 * np.cos(np.pi * ks / (n + 1))
    assert np.abs(np.sort(r.theta_all) - np.sort(lam)).max() <= 1e-13
    assert r.lanczos.beta[16] <= 1e-8


# ---------------------------------------------------------------- P16 (O3-O9, 2-D)
def test_p16_grid_dirichlet_closed_form():
    """5-point Dirichlet Laplacian on a 300 x 200 grid (the mesh class of C6): it is
    the Kronecker sum T_nx (+) T_ny, with eigenvectors sin(pi i x/(nx+1)) sin(pi j y/(ny+1))
    and eigenvalues 4 - 2cos(pi i/(nx+1)) - 2cos(pi j/(ny+1)). v1 = sum of 8 such modes
    with well-separated eigenvalues: the Krylov space is their span, so the 8 Ritz values
    are those eigenvalues (the P4 argument in two dimensions). Modes with clustered
    eigenvalues near the dense centre of this spectrum are avoided: there the rounding
    error of the sine vectors (~1e-16 along the other 59,992 modes) is amplified by the
    Krylov polynomial through small beta_i (measured: 12 modes including 3.9732/3.9739
    leave beta_13 = 3.6e-3 and Ritz values 2e-6 off)."""
    nx, ny = 300, 200
    A = S.grid_dirichlet(nx, ny)
    assert A.n == nx * ny and A.nnz == 5 * nx * ny - 2 * (nx + ny)
    modes = [(1, 1), (300, 200), (40, 30), (260, 170), (100, 60), (200, 140), (150, 100), (120, 40)]
    x = np.arange(1, nx + 1)
    y = np.arange(1, ny + 1)
    v1 = np.zeros(nx * ny)
    for i, j in modes:  # vertex r = (y-1) * nx + (x-1)
        v1 += np.outer(np.sin(np.pi * j * y / (ny + 1)), np.sin(np.pi * i * x / (nx + 1))).ravel()
    lam = np.array([4 - 2 * np.cos(np.pi * i / (nx + 1)) - 2 * np.cos(np.pi * j / (ny + 1)) for i, j in modes])
    assert np.min(np.diff(np.sort(lam))) > 1e-6
    r = O.solve(A.rowptr, A.col, A.val, K=8, m=8, v1vec=v1, tau=0.0, want_vectors=False)
    assert np.abs(np.sort(r.theta_all) - np.sort(lam)).max() <= 1e-12
    assert r.lanczos.beta[8] <= 1e-9


def test_grid_laplacian_generator_properties():
    """The weighted grid Laplacian D - W (C6 recipe): symmetric bit for bit, zero row
    sums, off-diagonals only between grid neighbours, and its kernel dimension equals
    the number of connected components of the kept edges (graph theory)."""
    nx, ny = 23, 17
    A = S.grid_laplacian(nx, ny, 0.35, 11)
    D = A.to_dense()
    assert np.array_equal(D, D.T) and np.abs(D.sum(axis=1)).max() == 0.0
    r, c = np.nonzero(D - np.diag(np.diag(D)))
    d = np.abs(r - c)
    assert np.all((d == 1) & (r // nx == c // nx) | (d == nx))
    import scipy.sparse.csgraph as cg
    ncomp, _ = cg.connected_components(sp.csr_matrix(D != 0))
    ev = np.linalg.eigvalsh(D)
    assert np.sum(np.abs(ev) <= 1e-10) == ncomp and ev.min() > -1e-10


# ---------------------------------------------------------------- P5, P7 (O4-O10)
@pytest.mark.parametrize("kind", ["dirichlet", "cycle"])
def test_p5_kahan_bound_random_start(kind):
    """Random v1: every Ritz value lies within its true residual of a closed-form
    eigenvalue (min_k |theta - lambda_k| <= ||A y - theta y||)."""
    n = 100_000
    A = S.dirichlet(n) if kind == "dirichlet" else S.cycle_laplacian(n)
    r = O.solve(A.rowptr, A.col, A.val, K=16, m=16, seed=9)
    kk = np.arange(1, n + 1) if kind == "dirichlet" else np.arange(n)
    lam = (2 - 2 * np.cos(np.pi * kk / (n + 1))) if kind == "dirichlet" else \
        (2 - 2 * np.cos(2 * np.pi * kk / n))
    lam = np.sort(lam)
    for t, y in zip(r.eigenvalues, r.eigenvectors):
        res = np.linalg.norm(O.spmv(A.rowptr, A.col, A.val, y) - t * y)
        i = np.searchsorted(lam, t)
        d = min(abs(lam[max(i - 1, 0)] - t), abs(lam[min(i, n - 1)] - t))
        assert d <= res * (1 + 1e-9) + 1e-14


@pytest.mark.parametrize("n", [6, 12, 13, 40, 64])
def test_p6_cycle_breakdown_and_multiplicity(n):
    """Cycle Laplacian: n//2+1 distinct eigenvalues 2-2cos(2 pi k/n); Lanczos from a
    generic v1 breaks down at exactly i = n//2 + 1 and its Ritz values are those."""
    A = S.cycle_laplacian(n)
    r = O.solve(A.rowptr, A.col, A.val, K=n, m=n, seed=4)
    distinct = np.unique(np.round(2 - 2 * np.cos(2 * np.pi * np.arange(n) / n), 12))
    assert r.lanczos.breakdown
    assert r.lanczos.m_found == n // 2 + 1 == len(distinct)
    assert np.allclose(np.sort(r.theta_all), distinct, atol=1e-12)


@pytest.mark.parametrize("m", [8, 24, 64])
def test_p7_lanczos_invariants(m):
    """Orthonormal basis, Lanczos relation, residual estimate = true residual,
    trace(T) = sum(theta), theta inside the spectrum bounds."""
    A = S.rmat(12, 40_000, 5)
    n = A.n
    rp, c, v = A.rowptr, A.col, A.val
    r = O.solve(rp, c, v, K=8, m=m, seed=2)
    lz = r.lanczos
    V = lz.V
    mf = lz.m_found
    assert np.abs(V @ V.T - np.eye(mf)).max() <= 1e-13
    M = sp.csr_matrix((v, c, rp), shape=(n, n))
    T = O.tridiag_dense(lz.alpha, lz.beta)
    AV = (M @ V.T)
    # residual of the Lanczos relation, using the next direction w = beta_{m+1} v_{m+1}
    R = AV - V.T @ T
    nrmA = spla.norm(M, 2) if n < 3000 else abs(spla.eigsh(M, 1, which="LM")[0][0])
    # all columns except the last satisfy the three-term relation exactly
    assert np.abs(R[:, :-1]).max() <= 1e-12 * nrmA
    assert abs(np.linalg.norm(R[:, -1]) - lz.beta[mf]) <= 1e-12 * nrmA
    for k, (t, y) in enumerate(zip(r.eigenvalues, r.eigenvectors)):
        true = np.linalg.norm(M @ y - t * y)
        assert abs(true - r.residual_est[k]) <= 1e-12 * nrmA
    assert abs(np.trace(T) - r.theta_all.sum()) <= 1e-12 * nrmA * m
    assert np.all(np.abs(r.theta_all) <= nrmA * (1 + 1e-12))


# ---------------------------------------------------------------- P15 (O8-O9 sign, reading Q12)


@pytest.mark.parametrize("case", ["rmat_m24", "er_m64", "two_by_two"])
def test_p15_ritz_sign_rule(case):
    """Reading Q12: each returned eigenvector y_k is unit-norm with <y_k, v1/||v1||> > 0.
    With an orthonormal basis, <y_k, v1> = |s_1k| where s_k is the unit eigenvector of T
    for theta_k; |s_1k| is sign-invariant, so it is taken from numpy.linalg.eigh(T)
    (LAPACK), not from the oracle's Jacobi. The inner products are formed here with
    numpy from the returned vectors and the start vector, not by the oracle. Each case
    also checks that the oracle's Jacobi hands back S[0,k] < 0 for at least one selected
    k, so the flip branch is exercised (a sign rule that never flips, or flips the wrong
    way, fails)."""
    if case == "rmat_m24":
        A = S.rmat(12, 40_000, 5)
        rp, c, v, K, m, seed = A.rowptr, A.col, A.val, 8, 24, 3
    elif case == "er_m64":
        rp, c, v = er_csr(2000, 12_000, 4)
        K, m, seed = 12, 64, 7
    else:
        rp, c, v = csr_of(np.array([[2.0, 1.0], [1.0, 2.0]]))
        K, m, seed = 2, 2, 1
    n = len(rp) - 1
    u = O.v1(seed, n)
    v1n = u / np.linalg.norm(u)
    r = O.solve(rp, c, v, K=K, m=m, seed=seed)
    T = O.tridiag_dense(r.lanczos.alpha, r.lanczos.beta)
    w, Q = np.linalg.eigh(T)
    flipped = 0
    for k in range(len(r.eigenvalues)):
        y = r.eigenvectors[k]
        assert abs(np.linalg.norm(y) - 1.0) <= 1e-12
        ip = float(np.dot(y, v1n))
        assert ip > 0.0, (case, k, ip)
        j = int(np.argmin(np.abs(w - r.eigenvalues[k])))
        assert abs(ip - abs(Q[0, j])) <= 1e-9, (case, k, ip, Q[0, j])
        flipped += r.S[0, r.idx[k]] < 0.0
    if case != "two_by_two":
        assert flipped >= 1, "no selected Jacobi column had S[0,k] < 0: the flip is untested"


# ---------------------------------------------------------------- P8 (O4-O9)
@pytest.mark.slow
def test_p8_converged_pairs_match_arpack():
    A = S.rmat(14, 120_000, 14)
    n = A.n
    M = sp.csr_matrix((A.val, A.col, A.rowptr), shape=(n, n))
    r = O.solve(A.rowptr, A.col, A.val, K=8, m=64, seed=1)
    ref = spla.eigsh(M, 8, which="LM", tol=1e-14)[0]
    ref = ref[np.argsort(-np.abs(ref))]
    nrm = abs(ref[0])
    conv = r.residual_est <= 1e-10 * nrm
    assert conv.sum() >= 4
    assert np.allclose(r.eigenvalues[conv], ref[conv], rtol=1e-10, atol=0)


# ---------------------------------------------------------------- P11 (adaptive stop)
def test_p11_adaptive_stop_kahan_and_minimal():
    """solve_adaptive (reading Q25): every returned pair satisfies the Kahan bound
    against dense eigenvalues (brute force), its explicit residual ||Ay - theta y||
    is within tol |theta_1|, and the previous check point had not converged
    (computed through plain solve at that m, not through the adaptive loop)."""
    A = S.rmat(11, 12_000, 5)
    n, K, tol, c = A.n, 6, 1e-7, 6
    lam = np.linalg.eigvalsh(dense(n, A.rowptr, A.col, A.val))
    r = O.solve_adaptive(A.rowptr, A.col, A.val, K, m_max=300, tol=tol, check=c, seed=2)
    assert r.extra["converged_stop"]
    i = r.lanczos.m_found
    assert i % c == 0 and K <= i < 300
    M = sp.csr_matrix((A.val, A.col, A.rowptr), shape=(n, n))
    t1 = abs(r.eigenvalues[0])
    for k in range(K):
        y = r.eigenvectors[k]
        true = np.linalg.norm(M @ y - r.eigenvalues[k] * y)
        assert true <= tol * t1 * (1 + 1e-6) + 1e-12 * t1
        assert np.min(np.abs(lam - r.eigenvalues[k])) <= true + 1e-12 * t1
    assert abs(t1 - np.abs(lam).max()) <= 1e-10 * t1
    if i - c >= K:
        prev = O.solve(A.rowptr, A.col, A.val, K, m=i - c, seed=2, want_vectors=False)
        assert np.any(prev.residual_est > tol * abs(prev.eigenvalues[0]))
    # a tolerance nothing meets runs to m_max
    r2 = O.solve_adaptive(A.rowptr, A.col, A.val, K, m_max=24, tol=1e-300, check=c, seed=2,
                          want_vectors=False)
    assert r2.lanczos.m_found == 24 and not r2.extra["converged_stop"]


# ---------------------------------------------------------------- P12 (thick restart)
def test_p12_thick_restart_relation_and_convergence():
    """solve_thick_restart (reading Q26): after restarts the basis stays
    orthonormal and the Lanczos relation A V_m = V_m T_m + beta v_{m+1} e_m^T
    holds with the arrowhead T (a wrong coupling b_j, sign or index breaks it);
    run to convergence, the K pairs match dense eigvalsh (brute force) and obey
    the Kahan bound; zero restarts is the plain solve."""
    A = S.rmat(11, 12_000, 5)
    n = A.n
    D = dense(n, A.rowptr, A.col, A.val)
    lam = np.linalg.eigvalsh(D)
    lam_top = lam[np.argsort(-np.abs(lam))]
    nrmA = np.abs(lam).max()
    K, m, keep = 6, 24, 12
    r = O.solve_thick_restart(A.rowptr, A.col, A.val, K, m, keep, max_restarts=3, seed=2)
    assert r.extra["restarts"] == 3 and r.extra["iterations"] == m + 3 * (m - keep)
    Vm, Tm, vn = r.lanczos.V, r.extra["T"], r.extra["v_next"]
    assert np.abs(Vm @ Vm.T - np.eye(m)).max() <= 1e-12
    assert abs(np.dot(Vm[0], vn)) <= 1e-12 and abs(np.linalg.norm(vn) - 1) <= 1e-12
    R = (D @ Vm.T) - Vm.T @ Tm
    R[:, m - 1] -= r.lanczos.beta[m] * vn
    assert np.abs(R).max() <= 1e-11 * nrmA
    assert np.count_nonzero(np.abs(Tm[:keep, :keep] - np.diag(np.diag(Tm[:keep, :keep]))) > 0) == 0
    # converged run
    rc = O.solve_thick_restart(A.rowptr, A.col, A.val, K, m, keep, max_restarts=50, tol=1e-10, seed=2)
    assert rc.extra["restarts"] < 50
    assert np.allclose(rc.eigenvalues, lam_top[:K], rtol=0, atol=1e-8 * nrmA)
    for kk in range(K):
        y = rc.eigenvectors[kk]
        true = np.linalg.norm(D @ y - rc.eigenvalues[kk] * y)
        assert np.min(np.abs(lam - rc.eigenvalues[kk])) <= true + 1e-12 * nrmA
    # no restart = the plain solve
    r0 = O.solve_thick_restart(A.rowptr, A.col, A.val, K, m, keep, max_restarts=0, seed=2)
    p = O.solve(A.rowptr, A.col, A.val, K, m=m, seed=2)
    assert np.allclose(np.sort(r0.theta_all), np.sort(p.theta_all), rtol=0, atol=1e-12 * nrmA)


# ---------------------------------------------------------------- P13 (periodic reorth)
def test_p13_periodic_reorth_special_cases():
    """solve_periodic (reading Q28): period 1 is the full-reorthogonalisation oracle
    bit for bit, a period beyond m is the no-reorthogonalisation oracle bit for bit,
    and period 4 (pairs of reorthogonalised iterations) keeps the basis orthogonal to
    1e-12 and the Ritz values within 1e-12 of full reorthogonalisation."""
    A = S.rmat(12, 30_000, 3)
    m, K = 40, 8
    full = O.solve(A.rowptr, A.col, A.val, K, m=m, seed=4, reorth=1)
    none = O.solve(A.rowptr, A.col, A.val, K, m=m, seed=4, reorth=0)
    p1 = O.solve_periodic(A.rowptr, A.col, A.val, K, m, 1, seed=4)
    pinf = O.solve_periodic(A.rowptr, A.col, A.val, K, m, m + 1, seed=4)
    assert np.array_equal(p1.theta_all, full.theta_all) and np.array_equal(p1.eigenvectors, full.eigenvectors)
    assert np.array_equal(pinf.theta_all, none.theta_all)
    p4 = O.solve_periodic(A.rowptr, A.col, A.val, K, m, 4, seed=4)
    orth = lambda V: np.abs(V @ V.T - np.eye(len(V))).max()
    assert orth(full.lanczos.V) <= 1e-13
    assert orth(p4.lanczos.V) <= 1e-12 < orth(none.lanczos.V)
    nrm = np.abs(full.theta_all).max()
    assert np.abs(np.sort(p4.theta_all) - np.sort(full.theta_all)).max() <= 1e-12 * nrm


# ---------------------------------------------------------------- P14 (partial reorth)
def test_p14_partial_reorth_keeps_semi_orthogonality():
    """solve_pro (reading Q29): Simon's estimate triggers reorthogonalisation of pairs
    of consecutive vectors; the basis stays semi-orthogonal (<= 10 sqrt(eps), what the
    scheme guarantees), the Ritz values equal the full-reorthogonalisation oracle to
    1e-12 |theta_1|, and only a fraction of the iterations pay for the pass."""
    A = S.rmat(12, 30_000, 3)
    m, K, eps = 48, 8, 2.0 ** -53
    full = O.solve(A.rowptr, A.col, A.val, K, m=m, seed=4, reorth=1)
    none = O.solve(A.rowptr, A.col, A.val, K, m=m, seed=4, reorth=0)
    p = O.solve_pro(A.rowptr, A.col, A.val, K, m, eps, seed=4)
    V = p.lanczos.V
    assert np.abs(V @ V.T - np.eye(m)).max() <= 10 * np.sqrt(eps)
    assert np.abs(none.lanczos.V @ none.lanczos.V.T - np.eye(m)).max() > 10 * np.sqrt(eps)
    nrm = np.abs(full.theta_all).max()
    assert np.abs(np.sort(p.theta_all) - np.sort(full.theta_all)).max() <= 1e-12 * nrm
    st = p.extra["reorth_steps"]
    assert 0 < len(st) < m // 2
    assert all(b == a + 1 for a, b in zip(st[0::2], st[1::2]))
