"""C-ABI boundary tests that need no GPU: the library loads, exports every
symbol include/topk_eig.h declares, plans partitions bit-exactly like the
oracle (rule P), and refuses to run without a B200."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, has_gpu

import oracle as O
import synthgen as S
import paper_2201_07498_b200 as T


def header_symbols():
    src = open(os.path.join(ROOT, "include", "topk_eig.h")).read()
    return sorted(set(re.findall(r"\b(topk_eig_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2201_07498_b200 as T
    lib = ctypes.CDLL(T.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    """The fatbinary carries sm_100a SASS (no PTX for JIT to other archs)."""
    import subprocess
    import paper_2201_07498_b200 as T
    out = subprocess.run(["cuobjdump", "--list-elf", T.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_plan_partition_matches_oracle(G):
    import paper_2201_07498_b200 as T
    for m in (S.rmat(14, 100_000, 3), S.dirichlet(1000), S.path_laplacian(77)):
        assert np.array_equal(T.plan_partition(m.rowptr, G), O.partition(m.rowptr, G))


def test_plan_partition_random_small_cases():
    import paper_2201_07498_b200 as T
    rng = np.random.default_rng(11)
    for _ in range(2000):
        n = int(rng.integers(1, 40))
        G = int(rng.integers(1, n + 1))
        rownnz = rng.integers(0, 9, n) * (rng.random(n) > 0.4)
        rp = np.concatenate([[0], np.cumsum(rownnz)]).astype(np.int64)
        assert np.array_equal(T.plan_partition(rp, G), O.partition(rp, G)), (rownnz, G)


def test_plan_partition_errors():
    import paper_2201_07498_b200 as T
    with pytest.raises(T.TopkError) as e:
        T.plan_partition(np.array([0, 1, 2]), 3)
    assert e.value.status == 1
    with pytest.raises(T.TopkError) as e:
        T.plan_partition(np.array([0, 2, 1]), 1)
    assert e.value.status == 2


@pytest.mark.skipif(has_gpu(), reason="checks the no-device path")
def test_create_without_gpu_fails_loudly():
    import paper_2201_07498_b200 as T
    A = S.dirichlet(100)
    with pytest.raises(T.TopkError) as e:
        T.TopkEig(A, 4, "f64", "f64")
    assert e.value.status == 8  # TOPK_E_NODEVICE: no CPU fallback


def test_create_argument_errors_precede_device():
    """Invalid arguments are rejected with E_INVALID/E_STRUCTURE/E_NOT_SYMMETRIC."""
    import paper_2201_07498_b200 as T
    A = S.dirichlet(50)
    for kw, st in [(dict(K=0), 1), (dict(K=51), 1), (dict(K=4, m=3), 1), (dict(K=4, parts=0), None)]:
        K = kw.pop("K")
        try:
            T.TopkEig(A, K, "f64", "f64", **kw).close()
        except T.TopkError as e:
            if st is not None:
                assert e.status == st
    bad = S.CSR(3, np.array([0, 1, 3, 2]), np.array([0, 1, 2], np.int32), np.ones(3))
    with pytest.raises(T.TopkError) as e:
        T.TopkEig(bad, 1, "f64", "f64")
    assert e.value.status == 2
    asym = S.from_dense(np.array([[1.0, 2.0], [0.0, 1.0]]))
    with pytest.raises(T.TopkError) as e:
        T.TopkEig(asym, 1, "f64", "f64")
    assert e.value.status == 3
    # thick restart / adaptive options (readings Q25, Q26)
    for kw in (dict(m=20, restart_keep=3), dict(m=20, restart_keep=19), dict(m=20, restart_keep=8, reorth=-1),
               dict(m=20, restart_keep=-1), dict(m=20, max_restarts=-2), dict(m=20, conv_tol=-1.0)):
        with pytest.raises(T.TopkError) as e:
            T.TopkEig(A, 4, "f64", "f64", **kw)
        assert e.value.status == 1, kw


# ---------------------------------------------------------------- host layout (no device)
@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("storage,dtype", [("f64", "f64"), ("f32", "f32"), ("f32", "bf16"), ("bf16", "bf16")])
def test_plan_layout_bit_exact_vs_oracle(G, storage, dtype):
    """Rows a3-a4: the library's host layout (what create
    uploads) equals the oracle's, bit for bit: degree row order, remapped
    columns, stored values."""
    A = S.rmat(13, 120_000, 5)  # long rows (> 2048 nnz) present
    b = O.partition(A.rowptr, G)
    for g in range(G):
        L = T.plan_layout(A, G, g, storage, dtype)
        orp, ocol, oval, onpad, operm = O.layout(A.rowptr, A.col, A.val, G, b, g, dtype, with_perm=True)
        assert L["n_pad"] == onpad
        assert np.array_equal(L["perm"], operm)
        assert np.array_equal(L["rowptr"], orp) and np.array_equal(L["col"], ocol)
        assert np.array_equal(L["val"].view(np.uint64), oval.view(np.uint64))


@pytest.mark.parametrize("G", [1, 2])
def test_plan_layout_parallel_degree_order_vs_oracle(G):
    """Parts with >= 2^16 rows take the multi-threaded counting sort (per-thread
    histograms over row chunks): same stable degree order as the oracle."""
    A = S.rmat(18, 1_200_000, 9)
    b = O.partition(A.rowptr, G)
    for g in range(G):
        assert b[g + 1] - b[g] >= 2 ** 16
        L = T.plan_layout(A, G, g, "f32", "f32")
        orp, ocol, oval, onpad, operm = O.layout(A.rowptr, A.col, A.val, G, b, g, "f32", with_perm=True)
        assert np.array_equal(L["perm"], operm)
        assert np.array_equal(L["rowptr"], orp) and np.array_equal(L["col"], ocol)


def test_csr_validation_and_canonicalisation_paths():
    """Row a1's one-pass CSR check (range, monotonic row pointers, strictly increasing
    columns): a canonical CSR is borrowed, a CSR with unsorted / duplicated columns in a
    row takes the regrouping path and lays out exactly like the oracle's canonical form
    (duplicates summed in input order), and malformed input is E_STRUCTURE."""
    A = S.rmat(12, 40_000, 3)
    rng = np.random.default_rng(1)
    col, val = A.col.copy(), A.val.copy()
    for r in rng.choice(A.n, 200, replace=False):  # shuffle some rows' entries
        a, b = A.rowptr[r], A.rowptr[r + 1]
        if b - a > 1:
            o = rng.permutation(b - a)
            col[a:b], val[a:b] = col[a:b][o], val[a:b][o]
    U = S.CSR(A.n, A.rowptr, col, val)
    rows = np.repeat(np.arange(A.n), np.diff(A.rowptr))
    crp, ccol, cval = O.coo_to_csr(A.n, rows, col, val)
    for G in (1, 2):
        b = O.partition(crp, G)
        for g in range(G):
            L = T.plan_layout(U, G, g, "f64")
            orp, ocol, oval, onpad = O.layout(crp, ccol, cval, G, b, g, "f64")
            assert np.array_equal(L["rowptr"], orp) and np.array_equal(L["col"], ocol)
            assert np.array_equal(L["val"].view(np.uint64), oval.view(np.uint64))
    # a duplicated entry inside a row (unsorted by equality): summed like COO
    r = int(np.argmax(np.diff(A.rowptr) > 2))
    a = A.rowptr[r]
    col2 = A.col.copy(); col2[a + 1] = col2[a]
    D = S.CSR(A.n, A.rowptr, col2, A.val)
    rp3, c3, v3 = O.coo_to_csr(A.n, rows, col2, A.val)
    L = T.plan_layout(D, 1, 0, "f64")
    orp, ocol, oval, _ = O.layout(rp3, c3, v3, 1, O.partition(rp3, 1), 0, "f64")
    assert np.array_equal(L["rowptr"], orp) and np.array_equal(L["col"], ocol)
    # malformed: column out of range, decreasing row pointer
    bad = A.col.copy(); bad[5] = A.n
    dec = A.rowptr.copy(); k = int(np.argmax(np.diff(A.rowptr) > 0)); dec[k + 1] = dec[k] - 1 if dec[k] > 0 else dec[k + 2] + 1
    for M in (S.CSR(A.n, A.rowptr, bad, A.val), S.CSR(A.n, dec, A.col, A.val)):
        with pytest.raises(T.TopkError) as e:
            T.plan_layout(M, 1, 0, "f64")
        assert e.value.status == 2


def test_host_block_cache_trim():
    """The create-time layout arrays (>= 1 MB) come from the library's host block cache
    (mem_pool.h): after a host-only layout the cached blocks are released by
    topk_eig_trim_pool, and a second trim finds nothing."""
    A = S.rmat(16, 500_000, 2)
    T.plan_layout(A, 1, 0, "f32")
    assert T.trim_pool() >= A.n * 4
    assert T.trim_pool() == 0


@pytest.mark.parametrize("G", [1, 3])
def test_physical_format_unpacks_to_logical(G):
    """The SpMV physical format (big-row CSR chunks + SELL-32 slices, host_prep.h)
    holds exactly the logical CSR: every logical entry at its physical slot,
    padding = (column 0, 0.0), slices degree-sorted, items cover all slices."""
    A = S.rmat(13, 120_000, 5)
    st = S.stars([8191, 8192, 8193, 16385, 300], dense=[127, 128, 129, 3])
    for M, g, G_ in [(A, g, G) for g in range(G)] + [(st, 0, 1)]:
        L = T.plan_layout(M, G_, g, "f32")
        rp, col, val, nbig, nne = L["rowptr"], L["col"], L["val"], L["nbig"], L["nnonempty"]
        deg = np.diff(rp)
        assert np.all(deg[:-1] >= deg[1:]), "rows must be in degree order"
        assert nne == int((deg > 0).sum()) and np.all(deg[:nbig] > 128) and np.all(deg[nbig:] <= 128)
        pcol, pval, ch, sl, it = L["pcol"], L["pval"], L["chunks"], L["sell"], L["items"]
        # big rows: CSR prefix, cut into <= 8192-nnz chunks (kChunkNnz) in order
        assert np.array_equal(pcol[:rp[nbig]], col[:rp[nbig]]) and np.array_equal(pval[:rp[nbig]], val[:rp[nbig]])
        cover = np.zeros(rp[nbig], np.int32)
        for row, z0, cnt, lid in ch:
            assert rp[row] <= z0 and z0 + cnt <= rp[row + 1] and 1 <= cnt <= 8192
            assert (lid >= 0) == (deg[row] > 8192)
            cover[z0:z0 + cnt] += 1
        assert np.all(cover == 1)
        # SELL-32: slice s rows nbig + 32 s + i, width = degree of its first row, column-major
        nsl = (nne - nbig + 31) // 32
        assert len(sl) == nsl
        seen = np.zeros(len(pcol), bool)
        seen[:rp[nbig]] = True
        for s_, (base, w) in enumerate(sl):
            p0 = nbig + 32 * s_
            assert w == deg[p0]
            for i in range(32):
                p = p0 + i
                d = deg[p] if p < nne else 0
                idx = base + 32 * np.arange(w) + i
                seen[idx] = True
                assert np.array_equal(pcol[idx[:d]], col[rp[p]:rp[p] + d]) if d else True
                assert np.array_equal(pval[idx[:d]], val[rp[p]:rp[p] + d]) if d else True
                assert np.all(pval[idx[d:]] == 0.0) and np.all(pcol[idx[d:]] == 0)
        assert seen.all()
        covered = np.concatenate([np.arange(a, b_) for a, b_ in it]) if len(it) else np.zeros(0, int)
        assert np.array_equal(covered, np.arange(nsl))



def _sym_ok(T, A):
    h = T.plan_symmetry(A, 0, A.n)  # the hash sums create uses (host-only, runs everywhere)
    return bool(h[0] == h[2] and h[1] == h[3])


def test_symmetry_check_hash_multiset():
    """Row a2 (reading Q17): the multiset-hash symmetry check accepts a symmetric
    R-MAT and rejects one-bit, one-entry and swapped-value perturbations of it, and
    agrees with the oracle's exact check (O1, a search per entry) on every case."""
    import paper_2201_07498_b200 as T
    A = S.rmat(13, 60_000, 7)
    assert _sym_ok(T, A) and O.is_symmetric(A.n, A.rowptr, A.col, A.val)

    def variant(kind):
        rp, col, val = A.rowptr.copy(), A.col.copy(), A.val.copy()
        r = int(np.argmax(np.diff(rp) > 3))
        k = int(rp[r]) + 1
        if kind == "bit":
            val[k] = np.nextafter(val[k], np.inf)
        elif kind == "swap":
            j = k + 1
            val[k], val[j] = val[j], val[k] + 1.0 / 128
        else:  # drop one off-diagonal entry
            col = np.delete(col, k)
            val = np.delete(val, k)
            rp = rp.copy()
            rp[r + 1:] -= 1
        return S.CSR(A.n, rp, col, val)

    for kind in ("bit", "swap", "drop"):
        V = variant(kind)
        assert not _sym_ok(T, V), kind
        assert not O.is_symmetric(V.n, V.rowptr, V.col, V.val), kind
    if not has_gpu():  # the same check inside create: rejected before any device work
        for kind in ("bit", "swap", "drop"):
            with pytest.raises(T.TopkError) as e:
                T.TopkEig(variant(kind), 4, "f64", "f64")
            assert e.value.status == 3, kind


def test_symmetry_check_adversarial_vs_exact_oracle():
    """Adversarial inputs for a multiset hash (reading Q17), each compared with the
    oracle's exact check: value swaps between the two triangles that keep every
    multiset statistic but one pairing, entries moved to the mirror position of
    another entry, sign flips, stored +0.0 vs -0.0 (bitwise check), and
    randomly perturbed small matrices (300 cases): the library's verdict equals the
    oracle's on every one."""
    import paper_2201_07498_b200 as T
    rng = np.random.default_rng(11)
    cases = []
    base = np.zeros((7, 7))
    for (i, j, v) in [(0, 1, 0.5), (0, 2, 0.75), (1, 3, 1.25), (2, 5, 0.5), (4, 6, 1.0), (3, 3, 2.0)]:
        base[i, j] = base[j, i] = v
    cases.append(base)
    t = base.copy(); t[0, 1], t[0, 2] = t[0, 2], t[0, 1]  # swap two upper values: lower unchanged
    cases.append(t)
    t = base.copy(); t[1, 0], t[2, 0] = 0.75, 0.5; t[0, 1], t[0, 2] = 0.75, 0.5  # consistent swap: symmetric
    cases.append(t)
    t = base.copy(); t[4, 6] = -1.0  # sign flip of one triangle
    cases.append(t)
    t = base.copy(); t[0, 1] = 0.0; t[0, 3] = 0.5  # an upper entry moved along its row
    cases.append(t)
    for _ in range(300):
        n = int(rng.integers(2, 9))
        a = np.zeros((n, n))
        for _ in range(int(rng.integers(1, 12))):
            i, j = rng.integers(0, n, 2)
            v = float(rng.integers(1, 4)) / 4
            a[i, j] = a[j, i] = v
        kind = rng.integers(0, 4)
        if kind == 1:  # perturb one stored entry
            nz = np.argwhere(a != 0)
            if len(nz):
                i, j = nz[rng.integers(len(nz))]
                a[i, j] = a[i, j] + 0.25
        elif kind == 2:  # move one entry to a fresh position
            nz = np.argwhere(a != 0)
            if len(nz):
                i, j = nz[rng.integers(len(nz))]
                v = a[i, j]; a[i, j] = 0.0
                a[int(rng.integers(0, n)), int(rng.integers(0, n))] = v
        elif kind == 3:  # transpose-mirror swap of two values
            nz = np.argwhere(np.triu(a, 1) != 0)
            if len(nz) >= 2:
                (i, j), (k, l) = nz[rng.choice(len(nz), 2, replace=False)]
                a[i, j], a[k, l] = a[k, l], a[i, j]
        cases.append(a)
    for a in cases:
        A = S.from_dense(a) if np.any(a) else None
        if A is None:
            continue
        assert _sym_ok(T, A) == O.is_symmetric(A.n, A.rowptr, A.col, A.val), a
    # stored entries that are +0.0 and -0.0 at mirrored positions: equal values, different bits
    Z = S.from_dense(base)
    for r, c, v in ((2, 5, -0.0), (5, 2, 0.0)):
        k = int(Z.rowptr[r]) + int(np.where(Z.col[Z.rowptr[r]:Z.rowptr[r + 1]] == c)[0][0])
        Z.val[k] = v
    assert _sym_ok(T, Z) == O.is_symmetric(Z.n, Z.rowptr, Z.col, Z.val) == False
