"""Seeded synthetic input generators (input infrastructure, no method arithmetic).

Shared by the oracle (``oracle/``) and the CUDA path (``paper_2201_07498_b200``)
as the ONE thing both sides may use. Every matrix is a pure function of its
arguments (counter-based hashing), so both sides see identical inputs.

Workload shapes follow the paper's evaluation set (Table I:
SuiteSparse graphs with 5-57M nnz and the GAP-kron R-MAT) and BASELINE.json's
configs; the exact recipes are in DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynthgen.so")
_SRC = os.path.join(_HERE, "synthgen.c")


def build(force: bool = False) -> str:
    """Compile libsynthgen.so with gcc (OpenMP) in-tree."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _SO + ".tmp", _SRC])
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Csr(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("rowptr", ctypes.POINTER(ctypes.c_int64)),
                ("col", ctypes.POINTER(ctypes.c_int32)),
                ("val", ctypes.POINTER(ctypes.c_double))]


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        lib.sg_rmat.restype = ctypes.POINTER(_Csr)
        lib.sg_rmat.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                ctypes.c_double, ctypes.c_double, ctypes.c_uint64]
        lib.sg_tridiag.restype = ctypes.POINTER(_Csr)
        lib.sg_tridiag.argtypes = [ctypes.c_int, ctypes.c_int64]
        lib.sg_grid2d.restype = ctypes.POINTER(_Csr)
        lib.sg_grid2d.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_double,
                                  ctypes.c_uint64]
        lib.sg_free.argtypes = [ctypes.POINTER(_Csr)]
        lib.sg_er_coo.restype = ctypes.c_int64
        lib.sg_er_coo.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.sg_hash3.restype = ctypes.c_uint64
        lib.sg_hash3.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib = lib
    return _lib


@dataclass
class CSR:
    """Host CSR matrix: int64 rowptr[n+1], int32 col[nnz], float64 val[nnz]."""
    n: int
    rowptr: np.ndarray
    col: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.rowptr))
        np.add.at(a, (rows, self.col), self.val)
        return a


@dataclass
class COO:
    n: int
    row: np.ndarray  # int64
    col: np.ndarray  # int32
    val: np.ndarray  # float64


def _take(p) -> CSR:
    if not p:
        raise MemoryError("synthgen: generation failed (bad arguments or out of memory)")
    c = p.contents
    n, nnz = int(c.n), int(c.nnz)
    try:
        rowptr = np.ctypeslib.as_array(c.rowptr, shape=(n + 1,)).copy()
        col = np.ctypeslib.as_array(c.col, shape=(max(nnz, 1),))[:nnz].copy()
        val = np.ctypeslib.as_array(c.val, shape=(max(nnz, 1),))[:nnz].copy()
    finally:
        _load().sg_free(p)
    return CSR(n, rowptr, col, val)


def rmat(scale: int, samples: int, seed: int, n: int | None = None,
         a: float = 0.57, b: float = 0.19, c: float = 0.19) -> CSR:
    """Graph500-parameter R-MAT, symmetric, deduplicated, no self loops,
    bf16-exact weights k/128 (k in [64,191]); ids scrambled, ids >= n rejected."""
    if n is None:
        n = 1 << scale
    return _take(_load().sg_rmat(scale, n, samples, a, b, c, seed))


def dirichlet(n: int) -> CSR:
    """tridiag(-1, 2, -1): eigenvalues 2 - 2 cos(pi k / (n+1)), k = 1..n."""
    return _take(_load().sg_tridiag(0, n))


def path_laplacian(n: int) -> CSR:
    """Path-graph Laplacian: eigenvalues 2 - 2 cos(pi k / n), k = 0..n-1."""
    return _take(_load().sg_tridiag(1, n))


def cycle_laplacian(n: int) -> CSR:
    """Cycle Laplacian (n >= 3): eigenvalues 2 - 2 cos(2 pi k / n), k = 0..n-1."""
    return _take(_load().sg_tridiag(2, n))


def grid_dirichlet(nx: int, ny: int) -> CSR:
    """5-point Dirichlet Laplacian on an nx x ny grid (row-major ids): eigenvalues
    4 - 2 cos(pi i / (nx+1)) - 2 cos(pi j / (ny+1)), i = 1..nx, j = 1..ny."""
    return _take(_load().sg_grid2d(0, nx, ny, 0.0, 0))


def grid_laplacian(nx: int, ny: int, drop: float, seed: int) -> CSR:
    """Weighted graph Laplacian D - W of an nx x ny 4-neighbour grid with each edge
    dropped with probability `drop` (mesh / road-network class of PAPER.md Table I);
    weights k/128, k in [64, 191]; row-major ids (spatial locality); isolated
    vertices are empty rows."""
    return _take(_load().sg_grid2d(1, nx, ny, drop, seed))


def er_coo(n: int, samples: int, seed: int) -> COO:
    """Random symmetric COO with duplicates, values U[-1,1) (both triangles)."""
    ri = np.empty(2 * samples, np.int64)
    ci = np.empty(2 * samples, np.int32)
    v = np.empty(2 * samples, np.float64)
    k = _load().sg_er_coo(n, samples, seed, ri.ctypes.data, ci.ctypes.data, v.ctypes.data)
    return COO(n, ri[:k].copy(), ci[:k].copy(), v[:k].copy())


def from_dense(a: np.ndarray) -> CSR:
    """CSR of the nonzeros of a small dense matrix (tests)."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    rows, cols = np.nonzero(a)
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, rows + 1, 1)
    rowptr = np.cumsum(rowptr)
    return CSR(n, rowptr, cols.astype(np.int32), a[rows, cols].copy())


def stars(degrees, dense=(), gap: int = 7, seed: int = 3) -> CSR:
    """Symmetric test matrix with rows of exactly the given degrees (SpMV layout
    boundaries): for each d in `degrees` a star (a centre row joined to d leaf rows of
    degree 1), for each s in `dense` a dense s x s block (rows of degree s); `gap`
    empty rows before every component and a ragged empty tail. Values k/128,
    k in [64, 191] (exact in bf16/f32/f64), drawn from a seeded numpy generator."""
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    r0 = 0
    for d in degrees:
        r0 += gap
        c = r0
        leaves = np.arange(c + 1, c + 1 + d)
        w = rng.integers(64, 192, size=d).astype(np.float64) / 128.0
        rows += [np.full(d, c), leaves]
        cols += [leaves, np.full(d, c)]
        vals += [w, w]
        r0 = c + 1 + d
    for sz in dense:
        r0 += gap
        w = rng.integers(64, 192, size=(sz, sz)).astype(np.float64) / 128.0
        w = np.triu(w) + np.triu(w, 1).T
        ii, jj = np.meshgrid(np.arange(sz), np.arange(sz), indexing="ij")
        rows.append((r0 + ii).ravel()); cols.append((r0 + jj).ravel()); vals.append(w.ravel())
        r0 += sz
    n = r0 + gap + 5
    row = np.concatenate(rows); col = np.concatenate(cols); val = np.concatenate(vals)
    key = row.astype(np.int64) * n + col
    o = np.argsort(key, kind="stable")
    rowptr = np.zeros(n + 1, np.int64)
    np.add.at(rowptr, row + 1, 1)
    return CSR(n, np.cumsum(rowptr), col[o].astype(np.int32), val[o])


_MAGIC = b"TKEVCSR1"


def save_csr(path: str, A: CSR) -> None:
    """Write A as one flat binary file (magic, n, nnz, int64 rowptr[n+1], int32
    col[nnz] padded to 8 bytes, float64 val[nnz]) through a temporary name, so
    readers never see a partial file (one process per GPU: rank 0 writes, the
    others map it; SURVEY L0 "TKEV cache")."""
    tmp = path + f".tmp{os.getpid()}"
    with open(tmp, "wb") as f:
        f.write(_MAGIC)
        f.write(np.array([A.n, A.nnz], np.int64).tobytes())
        np.ascontiguousarray(A.rowptr, np.int64).tofile(f)
        np.ascontiguousarray(A.col, np.int32).tofile(f)
        if A.nnz % 2:
            f.write(b"\0" * 4)
        np.ascontiguousarray(A.val, np.float64).tofile(f)
    os.replace(tmp, path)


def load_csr_mmap(path: str) -> CSR:
    """Map a save_csr file read-only: the arrays are views of the page cache, shared
    by every process that maps the same file (no per-process copy)."""
    head = np.fromfile(path, dtype=np.int64, count=3)
    if head[:1].tobytes() != _MAGIC:
        raise ValueError(f"{path}: not a save_csr file")
    n, nnz = int(head[1]), int(head[2])
    o = 24
    rowptr = np.memmap(path, np.int64, "r", offset=o, shape=(n + 1,))
    o += 8 * (n + 1)
    col = np.memmap(path, np.int32, "r", offset=o, shape=(max(nnz, 1),))[:nnz]
    o += 4 * nnz + (4 if nnz % 2 else 0)
    val = np.memmap(path, np.float64, "r", offset=o, shape=(max(nnz, 1),))[:nnz]
    return CSR(n, rowptr, col, val)


def hash3(s: int, a: int, b: int) -> int:
    return int(_load().sg_hash3(s, a, b))


# ----------------------------------------------------------------------------
# Named workloads (BASELINE.json configs).
def config_matrix(name: str):
    """Return the synthetic matrix of a named config.

    C1: ER n=10,000, 50,000 samples (nnz ~ 1e5 after duplicate summation), seed 1 (COO).
    C2D: Dirichlet tridiag n=1,000,000.   C2C: cycle Laplacian n=1,000,000.
    C3: R-MAT S=22 (n=4,194,304), 31,457,280 samples, seed 22 -> nnz ~ 60M.
    C3S: R-MAT S=16 (n=65,536), 491,520 samples, seed 16 (C3 shape, oracle-fast).
    C4: R-MAT ids over 2^27 rejected if >= n = 100,000,000, 1,410,000,000 samples,
        seed 27 -> nnz ~ 1.5e9 (host RAM ~45 GB while generating).
    C6: weighted Laplacian of a 4096 x 4096 grid, 25 % of edges dropped, seed 6 ->
        n = 16,777,216, nnz ~ 67M (mesh / road class of Table I, e.g. hugetrace-00020:
        16.0 M rows, 47.8 M nnz; row-major ids keep the spatial locality).
    C6S: the same recipe on a 300 x 200 grid, seed 6 (oracle-fast).
    C4X: R-MAT S=27, n = 2^27 (GAP-kron's n), 2.0e9 samples, seed 28 ->
        nnz ~ 2.2e9 > 2^31 (host RAM ~70 GB while generating).
    """
    if name == "C1":
        return er_coo(10_000, 50_000, 1)
    if name == "C2D":
        return dirichlet(1_000_000)
    if name == "C2C":
        return cycle_laplacian(1_000_000)
    if name == "C3":
        return rmat(22, 31_457_280, 22)
    if name == "C3S":
        return rmat(16, 491_520, 16)
    if name == "C4":
        return rmat(27, 1_410_000_000, 27, n=100_000_000)
    if name == "C6":
        return grid_laplacian(4096, 4096, 0.25, 6)
    if name == "C6S":
        return grid_laplacian(300, 200, 0.25, 6)
    if name == "C4X":
        return rmat(27, 2_000_000_000, 28)
    raise KeyError(name)
