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


# ---------------------------------------------------------------- host layout (no device)
@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("storage,dtype", [("f64", "f64"), ("f32", "f32"), ("f32", "bf16"), ("bf16", "bf16")])
def test_plan_layout_bit_exact_vs_oracle(G, storage, dtype):
    """Rows a3-a4: the library's host layout (what create
    uploads) equals the oracle's, bit for bit: hub-first row order, remapped
    columns with the hot bit, stored values and the SpMV tile table."""
    A = S.rmat(13, 120_000, 5)  # long rows (> 1024 nnz) present
    b = O.partition(A.rowptr, G)
    for g in range(G):
        rp, col, val, npad, tiles, perm = T.plan_layout(A, G, g, storage, dtype)
        orp, ocol, oval, onpad, operm = O.layout(A.rowptr, A.col, A.val, G, b, g, dtype, storage=storage,
                                                 with_perm=True)
        assert npad == onpad
        assert np.array_equal(perm, operm)
        assert np.array_equal(rp, orp) and np.array_equal(col, ocol)
        assert np.array_equal(val.view(np.uint64), oval.view(np.uint64))
        assert np.array_equal(tiles, O.tiles(orp, 1024))


def test_tile_table_properties():
    """Every nonzero of every non-empty row is covered exactly once; packed
    tiles hold whole rows and <= 1024 nonzeros; long rows are split in order."""
    A = S.rmat(13, 120_000, 5)
    rp = A.rowptr
    t = O.tiles(rp, 1024)
    nz_rows = np.flatnonzero(np.diff(rp) > 0)
    cover = np.zeros(rp[-1], np.int32)
    assert (t[:, 3] >= 0).any(), "fixture should contain long rows"
    for zb, cnt, jb, lid in t:
        assert 1 <= cnt <= 1024
        cover[zb:zb + cnt] += 1
        r = nz_rows[jb]
        if lid < 0:
            assert rp[r] == zb
            end = zb + cnt
            assert end in rp  # whole rows only
        else:
            assert rp[r] <= zb < rp[r + 1] and zb + cnt <= rp[r + 1]
    assert (cover == 1).all()
