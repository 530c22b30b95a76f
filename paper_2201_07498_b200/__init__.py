"""paper_2201_07498_b200 — B200-native Top-K sparse eigensolver hot path
(arXiv 2201.07498: Lanczos + Jacobi, mixed precision, nnz-partitioned rows).

This module is ONLY argument marshalling over the C ABI in include/topk_eig.h
(libtopk_eig.so, sm_100a CUDA kernels). Every step of the method runs in the
library's kernels; there is no CPU or PyTorch fallback: if the extension is
missing this import fails, and on a machine without a B200 ``TopkEig`` raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOPK_LIB", os.path.join(_HERE, "libtopk_eig.so"))  # TOPK_LIB: dev override

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python tools/build.py` "
                      "(nvcc, sm_100a). There is no fallback implementation.")

_lib = ctypes.CDLL(LIB_PATH)

DTYPES = {"f64": 0, "f32": 1, "bf16": 2}
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_STRUCTURE", 3: "E_NOT_SYMMETRIC", 4: "E_NOMEM",
          5: "E_CUDA", 6: "E_NCCL", 7: "E_STATE", 8: "E_NODEVICE"}


class TopkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"topk_eig {STATUS.get(status, status)}: {msg}")
        self.status = status


class _Matrix(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int), ("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("row_idx", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("values", ctypes.c_void_p),
                ("values_dtype", ctypes.c_int)]


class _Opts(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("krylov_dim", ctypes.c_int32),
                ("reorth", ctypes.c_int32), ("num_parts", ctypes.c_int32),
                ("device", ctypes.c_int32), ("check_symmetry", ctypes.c_int32),
                ("values_storage", ctypes.c_int32), ("use_graph", ctypes.c_int32),
                ("breakdown_tol", ctypes.c_double), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("profile", ctypes.c_int32), ("conv_tol", ctypes.c_double),
                ("conv_check", ctypes.c_int32), ("restart_keep", ctypes.c_int32),
                ("max_restarts", ctypes.c_int32), ("exchange", ctypes.c_int32),
                ("reorth_period", ctypes.c_int32), ("jacobi_path", ctypes.c_int32),
                ("jacobi_cluster", ctypes.c_int32), ("restart_loop", ctypes.c_int32),
                ("ritz_path", ctypes.c_int32), ("overlap", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("k_found", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("breakdown", ctypes.c_int32), ("jacobi_sweeps", ctypes.c_int32),
                ("jacobi_converged", ctypes.c_int32), ("num_parts", ctypes.c_int32),
                ("beta_next", ctypes.c_double), ("ms_solve", ctypes.c_double),
                ("bytes_model", ctypes.c_int64), ("gpu_launches", ctypes.c_int64),
                ("converged_stop", ctypes.c_int32), ("conv_checks", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("reorth_passes", ctypes.c_int32),
                ("ms_lanczos", ctypes.c_double), ("ms_jacobi", ctypes.c_double),
                ("ms_ritz", ctypes.c_double), ("bytes_nvlink", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P, _I32, _I64, _U64, _D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
_S = ctypes.c_int
_SIGS = {
    "topk_eig_create": (_S, [_P, _P, _I32, _S, _S, _P]),
    "topk_eig_solve": (_S, [_P, _U64, _P, _P, _P, _S, _P, _P]),
    "topk_eig_solve_async": (_S, [_P, _U64, _P, _P, _S]),
    "topk_eig_sync": (_S, [_P, _P]),
    "topk_eig_stream": (_P, [_P]),
    "topk_eig_kernel_times": (_S, [_P, _P, _P]),
    "topk_eig_destroy": (None, [_P]),
    "topk_eig_trim_pool": (ctypes.c_size_t, []),
    "topk_eig_plan_halo": (_S, [_P, _I32, _I32, _P, _P, _P]),
    "topk_eig_plan_symmetry": (_S, [_P, _I64, _I64, _P]),
    "topk_eig_last_error": (ctypes.c_char_p, []),
    "topk_eig_nccl_id": (_S, [_P]),
    "topk_eig_plan_partition": (_S, [_P, _I64, _I32, _P]),
    "topk_eig_plan_layout": (_S, [_P, _I32, _I32, _S, _S, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "topk_eig_export_partition": (_S, [_P, _P]),
    "topk_eig_export_layout": (_S, [_P, _I32, _P, _P, _P, _P, _P, _P]),
    "topk_eig_export_tridiag": (_S, [_P, _P, _P, _P, _P]),
    "topk_eig_export_basis": (_S, [_P, _I32, _P, _P]),
    "topk_eig_export_basis_raw": (_S, [_P, _I32, _P, _P]),
    "topk_eig_debug_spmv": (_S, [_P, _P, _P]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _check(status: int):
    if status != 0:
        raise TopkError(status, _lib.topk_eig_last_error().decode())


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def nccl_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.topk_eig_nccl_id(buf))
    return buf.raw


def trim_pool() -> int:
    """Return the library's cached device and host blocks (topk_eig_trim_pool)."""
    return int(_lib.topk_eig_trim_pool())


def plan_halo(A, G: int, g: int) -> dict:
    """Host-only halo plan of part g (topk_eig_plan_halo): owner offsets and owner
    positions of the remote entries the part's SpMV reads (exchange="halo")."""
    keep = []
    mat = _matrix(A, keep)
    nh = ctypes.c_int64()
    _check(_lib.topk_eig_plan_halo(ctypes.byref(mat), G, g, ctypes.byref(nh), None, None))
    off = np.zeros(G + 1, np.int64)
    pos = np.zeros(max(nh.value, 1), np.int32)
    _check(_lib.topk_eig_plan_halo(ctypes.byref(mat), G, g, ctypes.byref(nh), _ptr(off), _ptr(pos)))
    return {"n_halo": nh.value, "off": off, "pos": pos[:nh.value]}


def plan_symmetry(A, r0: int, r1: int) -> np.ndarray:
    """The four symmetry-check hash sums of rows [r0, r1) (topk_eig_plan_symmetry)."""
    keep = []
    mat = _matrix(A, keep)
    out = np.zeros(4, np.uint64)
    _check(_lib.topk_eig_plan_symmetry(ctypes.byref(mat), int(r0), int(r1), _ptr(out)))
    return out


def plan_partition(rowptr, G: int) -> np.ndarray:
    """Rule-P boundaries (host only, no device)."""
    rp = np.ascontiguousarray(rowptr, dtype=np.int64)
    b = np.zeros(G + 1, np.int64)
    _check(_lib.topk_eig_plan_partition(_ptr(rp), len(rp) - 1, G, _ptr(b)))
    return b


def _matrix(A, keep: list) -> "_Matrix":
    mat = _Matrix()
    mat.n = int(A.n)
    if hasattr(A, "rowptr"):
        rp = np.ascontiguousarray(A.rowptr, dtype=np.int64)
        keep.append(rp)
        mat.format, mat.row_ptr = 0, rp.ctypes.data
        mat.nnz = int(rp[-1])
    else:
        ri = np.ascontiguousarray(A.row, dtype=np.int64)
        keep.append(ri)
        mat.format, mat.row_idx = 1, ri.ctypes.data
        mat.nnz = len(ri)
    col = np.ascontiguousarray(A.col, dtype=np.int32)
    keep.append(col)
    mat.col_idx = col.ctypes.data
    if A.val is not None:
        val = np.ascontiguousarray(A.val)
        if val.dtype not in (np.float64, np.float32):
            val = val.astype(np.float64)
        keep.append(val)
        mat.values = val.ctypes.data
        mat.values_dtype = DTYPES["f32"] if val.dtype == np.float32 else DTYPES["f64"]
    return mat


def plan_layout(A, G: int, g: int, storage: str = "f64", values_storage: str | None = None) -> dict:
    """Host-only layout of part g of G (no device): the logical CSR in degree
    order (rowptr, col, val, perm, n_pad) and the SpMV physical format (pcol,
    pval, chunks [nchunks, 4], sell [nslices, 2], items [nitems, 2], nbig,
    nnonempty) -- exactly what topk_eig_create uploads."""
    keep = []
    mat = _matrix(A, keep)
    st, vs = DTYPES[storage], DTYPES[values_storage or storage]
    sz = np.zeros(9, np.int64)
    _check(_lib.topk_eig_plan_layout(ctypes.byref(mat), G, g, st, vs, _ptr(sz), *([None] * 9)))
    npad, nr, nz, nne, nbig, nch, nsl, nit, nph = (int(v) for v in sz)
    out = dict(n_pad=npad, nnonempty=nne, nbig=nbig,
               rowptr=np.zeros(nr + 1, np.int64), col=np.zeros(max(nz, 1), np.int32),
               val=np.zeros(max(nz, 1)), perm=np.zeros(max(nr, 1), np.int32),
               pcol=np.zeros(max(nph, 1), np.int32), pval=np.zeros(max(nph, 1)),
               chunks=np.zeros((max(nch, 1), 4), np.int64), sell=np.zeros((max(nsl, 1), 2), np.int64),
               items=np.zeros((max(nit, 1), 2), np.int32))
    _check(_lib.topk_eig_plan_layout(ctypes.byref(mat), G, g, st, vs, None, *[_ptr(out[k]) for k in (
        "rowptr", "col", "val", "perm", "pcol", "pval", "chunks", "sell", "items")]))
    for k, m in (("col", nz), ("val", nz), ("perm", nr), ("pcol", nph), ("pval", nph), ("chunks", nch),
                 ("sell", nsl), ("items", nit)):
        out[k] = out[k][:m]
    return out


@dataclass
class Result:
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray | None
    residual_est: np.ndarray
    info: dict


class TopkEig:
    """Handle over topk_eig_create / topk_eig_solve.

    A: object with n, rowptr, col, val (CSR, e.g. synthgen.CSR) or n, row, col, val
    (COO). storage/compute: "f64" | "f32" | "bf16" (compute: "f64" | "f32").
    """

    def __init__(self, A, K: int, storage: str = "f32", compute: str = "f64", m: int | None = None,
                 reorth: int = 1, parts: int = 1, device: int = 0, check_symmetry: bool = True,
                 values_storage: str | None = None, use_graph: bool = True,
                 breakdown_tol: float = 0.0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, profile: bool = False,
                 conv_tol: float = 0.0, conv_check: int = 0, restart_keep: int = 0,
                 max_restarts: int = 0, exchange: str = "allgather", reorth_period: int = 0,
                 jacobi_path: str = "auto", jacobi_cluster: int = 0, restart_loop: str = "auto",
                 ritz_path: str = "auto", overlap: int = 0):
        self._h = ctypes.c_void_p()
        self.n = int(A.n)
        self.K = int(K)
        keep = []
        mat = _matrix(A, keep)
        o = _Opts()
        o.struct_size = ctypes.sizeof(_Opts)
        o.krylov_dim = int(m or 0)
        o.reorth = int(reorth)
        o.num_parts = int(parts)
        o.device = int(device)
        o.check_symmetry = 0 if check_symmetry else -1
        o.values_storage = DTYPES[values_storage] if values_storage else 0
        o.use_graph = 0 if use_graph else -1
        o.breakdown_tol = float(breakdown_tol)
        o.rank, o.world = int(rank), int(world)
        o.profile = 1 if profile else 0
        o.conv_tol = float(conv_tol)
        o.conv_check = int(conv_check)
        o.restart_keep = int(restart_keep)
        o.max_restarts = int(max_restarts)
        o.exchange = {"allgather": 0, "halo": 1}[exchange]
        o.reorth_period = int(reorth_period)
        o.jacobi_path = {"auto": 0, "single": 1, "cluster": 2}[jacobi_path]
        o.jacobi_cluster = int(jacobi_cluster)
        o.restart_loop = {"auto": 0, "unrolled": 1}[restart_loop]
        o.ritz_path = {"auto": 0, "cuda_cores": 1}[ritz_path]
        o.overlap = int(overlap)
        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
        _check(_lib.topk_eig_create(ctypes.byref(self._h), ctypes.byref(mat), self.K,
                                    DTYPES[storage], DTYPES[compute], ctypes.byref(o)))
        self.m = int(m or K)
        self.parts = int(parts)

    # ---- solve -------------------------------------------------------------
    def solve(self, seed: int = 1, v1=None, vectors: bool = True, vec_dtype: str = "f64") -> Result:
        ev = np.full(self.K, np.nan)
        rs = np.full(self.K, np.nan)
        Y = None
        if vectors:
            Y = np.zeros((self.K, self.n), np.float64 if vec_dtype == "f64" else np.float32)
        v1a = None if v1 is None else np.ascontiguousarray(v1, dtype=np.float64)
        info = Info()
        _check(_lib.topk_eig_solve(self._h, int(seed), _ptr(v1a), _ptr(ev), _ptr(Y),
                                   DTYPES[vec_dtype], _ptr(rs), ctypes.byref(info)))
        kf = info.k_found
        return Result(ev, None if Y is None else Y[:kf], rs, info.as_dict())

    def solve_async(self, seed: int, evals_dev_ptr: int, evecs_dev_ptr: int | None,
                    vec_dtype: str = "f32"):
        _check(_lib.topk_eig_solve_async(self._h, int(seed), evals_dev_ptr, evecs_dev_ptr,
                                         DTYPES[vec_dtype]))

    def sync(self) -> dict:
        info = Info()
        _check(_lib.topk_eig_sync(self._h, ctypes.byref(info)))
        return info.as_dict()

    KERNEL_CLASSES = ("v1", "spmv", "step", "correct", "jacobi", "ritz_norms", "ritz_out", "unperm")

    def kernel_times(self) -> dict:
        """{class: (total ms, launches)} of the last solve (profile=True)."""
        ms = np.zeros(8)
        n = np.zeros(8, np.int32)
        _check(_lib.topk_eig_kernel_times(self._h, _ptr(ms), _ptr(n)))
        return {c: (float(ms[i]), int(n[i])) for i, c in enumerate(self.KERNEL_CLASSES)}

    @property
    def stream(self) -> int:
        return int(_lib.topk_eig_stream(self._h) or 0)

    # ---- exports -----------------------------------------------------------
    def partition(self) -> np.ndarray:
        b = np.zeros(self.parts + 1, np.int64)
        _check(_lib.topk_eig_export_partition(self._h, _ptr(b)))
        return b

    def layout(self, part: int = 0):
        npad, nr, nz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.topk_eig_export_layout(self._h, part, None, None, None, ctypes.byref(npad),
                                           ctypes.byref(nr), ctypes.byref(nz)))
        rp = np.zeros(nr.value + 1, np.int64)
        c = np.zeros(max(nz.value, 1), np.int32)
        v = np.zeros(max(nz.value, 1), np.float64)
        _check(_lib.topk_eig_export_layout(self._h, part, _ptr(rp), _ptr(c), _ptr(v), None, None, None))
        return rp, c[:nz.value], v[:nz.value], npad.value

    def tridiag(self):
        mf = ctypes.c_int32()
        _check(_lib.topk_eig_export_tridiag(self._h, None, None, None, ctypes.byref(mf)))
        mm = mf.value
        a, b, t = np.zeros(max(mm, 1)), np.zeros(mm + 1), np.zeros(max(mm, 1))
        _check(_lib.topk_eig_export_tridiag(self._h, _ptr(a), _ptr(b), _ptr(t), None))
        return a[:mm], b, t[:mm]

    def basis(self, part: int = 0, raw: bool = False) -> np.ndarray:
        """Stored basis of `part` (part-local rows, original order): the normalised
        v_j (topk_eig_export_basis), or with raw=True the unscaled stored u_j
        (topk_eig_export_basis_raw; column 0 = the unnormalised start vector)."""
        fn = _lib.topk_eig_export_basis_raw if raw else _lib.topk_eig_export_basis
        nc = ctypes.c_int32()
        _check(fn(self._h, part, None, ctypes.byref(nc)))
        rp, _c, _v, _np = self.layout(part)
        nrows = len(rp) - 1
        V = np.zeros((nc.value, nrows), np.float64)
        _check(fn(self._h, part, _ptr(V), None))
        return V

    def debug_spmv(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.n, np.float64)
        _check(_lib.topk_eig_debug_spmv(self._h, _ptr(x), _ptr(y)))
        return y

    def close(self):
        if self._h:
            _lib.topk_eig_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def solve(A, K: int, **kw) -> Result:
    """One-shot create + solve."""
    solve_kw = {k: kw.pop(k) for k in ("seed", "v1", "vectors", "vec_dtype") if k in kw}
    with TopkEig(A, K, **kw) as h:
        return h.solve(**solve_kw)
