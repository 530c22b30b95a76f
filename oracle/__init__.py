"""Python front of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu_baseline / ``--impl reference`` legs may import this package.
The product path (paper_2201_07498_b200) never imports it and shares no code
with it. Arithmetic lives in oracle.c (plain single-threaded fp64 C, every
function citing PAPER.md); this file only marshals arrays and strings the C
steps together in the paper's order (Lanczos, then Jacobi on
T, then the Ritz projection 𝒱V).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

# breakdown thresholds tau per storage dtype (reading Q7)
TAU = {"f64": 1e-12, "f32": 1e-6, "bf16": 1e-3}
_DT = {"f64": 0, "f32": 1, "bf16": 2}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc: -O2, no -ffast-math (IEEE semantics kept),
    single-threaded, no vector intrinsics."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
                               "-shared", "-std=c11", "-o", _SO + ".tmp", _SRC, "-lm"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None
P = ctypes.c_void_p
I64, I32, U64, D = ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        sig = {
            "orc_coo_to_csr": (I64, [I64, I64, P, P, P, P, P, P]),
            "orc_is_symmetric": (ctypes.c_int, [I64, P, P, P]),
            "orc_partition": (ctypes.c_int, [I64, P, I32, P]),
            "orc_positions": (ctypes.c_int, [I64, P, I32, P, P]),
            "orc_layout": (I64, [I64, P, P, P, I32, P, I32, ctypes.c_int, P, P, P, P, P]),
            "orc_v1": (None, [U64, I64, P]),
            "orc_spmv": (None, [I64, P, P, P, P, P]),
            "orc_lanczos": (I64, [I64, P, P, P, P, I32, I32, D, P, P, P, P]),
            "orc_lanczos_iter": (ctypes.c_int, [I64, P, P, P, I32, I32, D, P, P, P, P, P, P]),
            "orc_jacobi": (ctypes.c_int, [I32, P, P, P, I32, P]),
            "orc_select": (I32, [I32, P, I32, P]),
            "orc_ritz": (None, [I64, I32, P, P, I32, P, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ---------------------------------------------------------------------------
def coo_to_csr(n, row, col, val):
    """O1: canonical CSR (rows grouped, columns sorted, duplicates summed in input order)."""
    row, col, val = _c(row, np.int64), _c(col, np.int32), _c(val, np.float64)
    nnz = len(val)
    rp = np.zeros(n + 1, np.int64)
    c = np.zeros(max(nnz, 1), np.int32)
    v = np.zeros(max(nnz, 1), np.float64)
    k = _load().orc_coo_to_csr(n, nnz, _p(row), _p(col), _p(val), _p(rp), _p(c), _p(v))
    if k < 0:
        raise ValueError(f"oracle coo_to_csr: error {-k}")
    return rp, c[:k].copy(), v[:k].copy()


def canonicalize_csr(n, rowptr, col, val):
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))
    return coo_to_csr(n, rows, col, val)


def is_symmetric(n, rowptr, col, val) -> bool:
    rowptr, col, val = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    return bool(_load().orc_is_symmetric(n, _p(rowptr), _p(col), _p(val)))


def partition(rowptr, G: int) -> np.ndarray:
    """O2: rule P boundaries b[0..G]."""
    rowptr = _c(rowptr, np.int64)
    n = len(rowptr) - 1
    b = np.zeros(G + 1, np.int64)
    if _load().orc_partition(n, _p(rowptr), G, _p(b)) != 0:
        raise ValueError("oracle partition: invalid G")
    return b


def positions(rowptr, G: int, b) -> np.ndarray:
    """Degree-order position of every row inside its part."""
    rowptr, b = _c(rowptr, np.int64), _c(b, np.int64)
    n = len(rowptr) - 1
    pos = np.zeros(max(n, 1), np.int32)
    _load().orc_positions(n, _p(rowptr), G, _p(b), _p(pos))
    return pos[:n]


def layout(rowptr, col, val, G: int, b, g: int, dtype: str = "f64", with_perm: bool = False):
    """O2: per-partition local CSR (degree row order, rebased rowptr, columns
    remapped into the padded replica, values rounded to dtype, returned as f64)
    and n_pad; with_perm: also return the position -> original row map."""
    rowptr, col, val, b = (_c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64),
                           _c(b, np.int64))
    n = len(rowptr) - 1
    pos = positions(rowptr, G, b)
    ng = int(b[g + 1] - b[g])
    zg = int(rowptr[b[g + 1]] - rowptr[b[g]])
    lrp = np.zeros(ng + 1, np.int64)
    lc = np.zeros(max(zg, 1), np.int32)
    lv = np.zeros(max(zg, 1), np.float64)
    perm = np.zeros(max(ng, 1), np.int32)
    npad = _load().orc_layout(n, _p(rowptr), _p(col), _p(val), G, _p(b), g, _DT[dtype], _p(pos),
                              _p(lrp), _p(lc), _p(lv), _p(perm))
    out = (lrp, lc[:zg].copy(), lv[:zg].copy(), int(npad))
    return out + (perm[:ng].copy(),) if with_perm else out


def v1(seed: int, n: int) -> np.ndarray:
    """O3: unnormalised start vector u_r = 2 U(h3(seed, 0x7631, r)) - 1."""
    u = np.zeros(n, np.float64)
    _load().orc_v1(seed, n, _p(u))
    return u


def spmv(rowptr, col, val, x) -> np.ndarray:
    rowptr, col, val, x = (_c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64),
                           _c(x, np.float64))
    n = len(rowptr) - 1
    y = np.zeros(n, np.float64)
    _load().orc_spmv(n, _p(rowptr), _p(col), _p(val), _p(x), _p(y))
    return y


@dataclass
class LanczosOut:
    alpha: np.ndarray      # alpha_1..alpha_m'
    beta: np.ndarray       # beta_1(=0)..beta_{m'+1}
    V: np.ndarray | None   # (m', n)
    m_found: int
    breakdown: bool


def lanczos(rowptr, col, val, v1vec, m: int, reorth: int = 1, tau: float = 1e-12,
            keep_V: bool = True) -> LanczosOut:
    rowptr, col, val, v1vec = (_c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64),
                               _c(v1vec, np.float64))
    n = len(rowptr) - 1
    alpha = np.zeros(m, np.float64)
    beta = np.zeros(m + 1, np.float64)
    V = np.zeros((m, n), np.float64) if keep_V else None
    bd = np.zeros(1, np.int32)
    mf = _load().orc_lanczos(n, _p(rowptr), _p(col), _p(val), _p(v1vec), m, reorth, tau,
                             _p(alpha), _p(beta), _p(V) if keep_V else None, _p(bd))
    if mf < 0:
        raise MemoryError("oracle lanczos: out of memory")
    return LanczosOut(alpha[:mf].copy(), beta[:mf + 1].copy(),
                      V[:mf].copy() if keep_V else None, int(mf), bool(bd[0]))


class LanczosRun:
    """Iteration-by-iteration driver over orc_lanczos_iter (the same arithmetic
    as orc_lanczos); used to time bounded samples of the oracle. Restarts from
    v1 after m iterations so the per-step reorth cost averages like a full solve."""

    def __init__(self, rowptr, col, val, v1vec, m: int, reorth: int = 1, tau: float = 1e-12):
        self.rp, self.c, self.v = (_c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64))
        self.n = len(self.rp) - 1
        self.m, self.reorth, self.tau = m, reorth, tau
        u = _c(v1vec, np.float64)
        self.v1 = u / np.sqrt(np.add.accumulate(u * u)[-1])  # sequential sum, as in oracle.c
        self.V = np.zeros((m, self.n))
        self.vt = np.zeros(self.n)
        self.vn = np.zeros(self.n)
        self.alpha = np.zeros(m)
        self.beta = np.zeros(m + 1)
        self.ts = np.zeros(1)
        self.i = 0

    def step(self) -> int:
        if self.i == self.m:
            self.i = 0
        if self.i == 0:
            self.V[0] = self.v1
            self.beta[0] = 0.0
            self.ts[0] = 0.0
        self.i += 1
        return _load().orc_lanczos_iter(self.n, _p(self.rp), _p(self.c), _p(self.v), self.i,
                                        self.reorth, self.tau, _p(self.V), _p(self.vt),
                                        _p(self.vn), _p(self.alpha), _p(self.beta), _p(self.ts))


def tridiag_dense(alpha, beta) -> np.ndarray:
    """O6: T = tridiag(beta_2..beta_m'; alpha_1..alpha_m'; beta_2..beta_m') (reading Q1)."""
    mm = len(alpha)
    T = np.diag(np.asarray(alpha, np.float64))
    for k in range(1, mm):
        T[k - 1, k] = T[k, k - 1] = beta[k]
    return T


def jacobi(A, max_sweeps: int = 50):
    """O7: cyclic Jacobi; returns (theta, S (columns = eigenvectors), sweeps, converged)."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    mm = A.shape[0]
    theta = np.zeros(mm, np.float64)
    S = np.zeros((mm, mm), np.float64)
    sw = np.zeros(1, np.int32)
    conv = _load().orc_jacobi(mm, _p(A), _p(theta), _p(S), max_sweeps, _p(sw))
    return theta, S, int(sw[0]), bool(conv)


def select(theta, K: int) -> np.ndarray:
    """O8: indices of the top-K by (-|theta|, -theta)."""
    theta = _c(theta, np.float64)
    idx = np.zeros(max(K, 1), np.int32)
    k = _load().orc_select(len(theta), _p(theta), K, _p(idx))
    return idx[:k].copy()


def ritz(V, S, idx) -> np.ndarray:
    """O9: normalised, sign-fixed Ritz vectors (K, n)."""
    V = _c(V, np.float64)
    S = _c(S, np.float64)
    idx = _c(idx, np.int32)
    mm, n = V.shape
    K = len(idx)
    Y = np.zeros((K, n), np.float64)
    _load().orc_ritz(n, mm, _p(V), _p(S), K, _p(idx), _p(Y))
    return Y


@dataclass
class SolveOut:
    eigenvalues: np.ndarray          # top-K' Ritz values, (-|θ|, -θ) order
    eigenvectors: np.ndarray | None  # (K', n)
    theta_all: np.ndarray            # all m' Ritz values (Jacobi order)
    S: np.ndarray
    idx: np.ndarray
    lanczos: LanczosOut
    jacobi_sweeps: int
    jacobi_converged: bool
    residual_est: np.ndarray         # |beta_{m'+1} s_{m',k}| for the selected k
    extra: dict = field(default_factory=dict)


def solve(rowptr, col, val, K: int, m: int | None = None, seed: int = 1, v1vec=None,
          reorth: int = 1, tau: float = 1e-12, want_vectors: bool = True) -> SolveOut:
    """The whole method in the paper's order:
    O3 v1 -> O4-O6 Lanczos -> O7 Jacobi on T -> O8 select -> O9 Ritz."""
    n = len(rowptr) - 1
    if m is None:
        m = K
    if v1vec is None:
        v1vec = v1(seed, n)
    lz = lanczos(rowptr, col, val, v1vec, m, reorth, tau, keep_V=want_vectors)
    T = tridiag_dense(lz.alpha, lz.beta)
    theta, S, sw, conv = jacobi(T)
    idx = select(theta, K)
    evals = theta[idx]
    Y = ritz(lz.V, S, idx) if want_vectors else None
    mm = lz.m_found
    rest = np.abs(lz.beta[mm] * S[mm - 1, idx]) if mm > 0 else np.zeros(0)
    return SolveOut(evals, Y, theta, S, idx, lz, sw, conv, rest)


def solve_adaptive(rowptr, col, val, K: int, m_max: int, tol: float, check: int | None = None,
                   seed: int = 1, v1vec=None, reorth: int = 1, tau: float = 1e-12,
                   want_vectors: bool = True) -> SolveOut:
    """Convergence-driven Krylov dimension (reading Q25).
    The paper runs a fixed number of iterations (Alg.1 l.3); this mode stops at the
    first check point i = c, 2c, ... (c = check or K) with K <= i < m_max and
    i <= m' (the iterations completed) where the K selected Ritz pairs of T_i all
    have residual estimate |beta_{i+1} s_{i,k}| <= tol |theta_1| (O10, reading Q6),
    and returns the solve at m = i. The first i Lanczos steps do not depend on how
    many follow, so the run to m_max is truncated at i (plain definition)."""
    n = len(rowptr) - 1
    if v1vec is None:
        v1vec = v1(seed, n)
    lz = lanczos(rowptr, col, val, v1vec, m_max, reorth, tau, keep_V=want_vectors)
    c = check or K
    stop = None
    i = c
    while i < m_max and i <= lz.m_found:
        if i >= K:
            theta, S, _, _ = jacobi(tridiag_dense(lz.alpha[:i], lz.beta[:i + 1]))
            idx = select(theta, K)
            res = np.abs(lz.beta[i] * S[i - 1, idx])
            if len(idx) == K and bool(np.all(res <= tol * abs(theta[idx[0]]))):
                stop = i
                break
        i += c
    if stop is not None:
        lz = LanczosOut(lz.alpha[:stop].copy(), lz.beta[:stop + 1].copy(),
                        None if lz.V is None else lz.V[:stop].copy(), stop, False)
    T = tridiag_dense(lz.alpha, lz.beta)
    theta, S, sw, conv = jacobi(T)
    idx = select(theta, K)
    Y = ritz(lz.V, S, idx) if want_vectors else None
    mm = lz.m_found
    rest = np.abs(lz.beta[mm] * S[mm - 1, idx]) if mm > 0 else np.zeros(0)
    return SolveOut(theta[idx], Y, theta, S, idx, lz, sw, conv, rest,
                    extra={"converged_stop": stop is not None})


def solve_thick_restart(rowptr, col, val, K: int, m: int, keep: int, max_restarts: int,
                        tol: float = 0.0, seed: int = 1, v1vec=None, tau: float = 1e-12,
                        want_vectors: bool = True) -> SolveOut:
    """Thick-restart Lanczos (Wu & Simon, SIAM J. Matrix Anal. Appl. 22(2), 2000;
    SURVEY 8(f) NEXT-2, reading Q26) around the paper's iteration
    (Alg.1 l.5-18 with full MGS reorthogonalisation, O4-O5) and Jacobi (O7):
      cycle: Lanczos steps i = k+1 .. m on V (k = 0 in the first cycle);
      end of cycle: T_m = S diag(theta) S^T (O7); stop if max_restarts restarts
        were done, or (tol > 0) all K selected pairs (O8) have residual estimate
        |beta_{m+1} s_{m,k}| <= tol |theta_1| (O10);
      restart: keep the `keep` Ritz pairs of largest |theta| (order O8):
        V[0:keep] = (V_m S_J)^T, V[keep] = v_{m+1},
        T = [[diag(theta_J), b], [b^T, .]] with b_j = beta_{m+1} s_{m,j};
        the first step after a restart subtracts sum_j b_j y_j instead of the
        beta_i v_{i-1} term (the arrowhead coupling), then MGS as usual.
    Plain numpy vector algebra + the oracle's C SpMV, fp64, no blocking."""
    n = len(rowptr) - 1
    if v1vec is None:
        v1vec = v1(seed, n)
    u = np.asarray(v1vec, np.float64)
    V = np.zeros((m + 1, n), np.float64)
    V[0] = u / np.sqrt(np.dot(u, u))
    T = np.zeros((m, m), np.float64)
    k = 0
    restarts = 0
    total = 0
    tscale = 0.0
    breakdown = False
    mm = m
    beta_next = 0.0
    while True:
        for i in range(k, m):                       # column i holds v_{i+1}
            y = spmv(rowptr, col, val, V[i])        # l.9
            a = float(np.dot(V[i], y))              # l.10
            T[i, i] = a
            tscale = max(tscale, abs(a))
            w = y - a * V[i]                        # l.11
            if i > k:
                w -= T[i, i - 1] * V[i - 1]
            elif k > 0:                             # first step after a restart
                for j in range(k):
                    w -= T[j, k] * V[j]
            for j in range(i + 1):                  # l.12-18 full reorth (MGS, Q3)
                w -= np.dot(V[j], w) * V[j]
            b = float(np.sqrt(np.dot(w, w)))        # l.6
            total += 1
            if i + 1 < m:
                if b <= tau * tscale:               # Q7
                    breakdown = True
                    mm = i + 1
                    beta_next = b
                    break
                T[i + 1, i] = T[i, i + 1] = b
                tscale = max(tscale, b)
            V[i + 1] = w / b                        # l.7
            beta_next = b
        Tm = T[:mm, :mm]
        theta, S, sw, conv = jacobi(Tm)
        idx = select(theta, K)
        res = np.abs(beta_next * S[mm - 1, idx])
        done = breakdown or restarts == max_restarts or (
            tol > 0 and len(idx) == K and bool(np.all(res <= tol * abs(theta[idx[0]]))))
        if done:
            break
        J = select(theta, keep)
        Y = S[:, J].T @ V[:m]                       # Ritz vectors (O9 without normalisation)
        bvec = beta_next * S[m - 1, J]
        V[keep] = V[m]
        V[:keep] = Y
        T = np.zeros((m, m), np.float64)
        for j in range(keep):
            T[j, j] = theta[J[j]]
            T[j, keep] = T[keep, j] = bvec[j]
        k = keep
        restarts += 1
    Y = ritz(V[:mm], S, idx) if want_vectors else None
    lz = LanczosOut(np.diag(Tm).copy(), np.zeros(mm + 1), V[:mm].copy(), mm, breakdown)
    lz.beta[mm] = beta_next
    return SolveOut(theta[idx], Y, theta, S, idx, lz, sw, conv, res,
                    extra={"restarts": restarts, "iterations": total, "T": Tm.copy(),
                           "v_next": V[mm].copy() if mm < m + 1 else None})


def solve_periodic(rowptr, col, val, K: int, m: int, period: int, seed: int = 1, v1vec=None,
                   tau: float = 1e-12, want_vectors: bool = True) -> SolveOut:
    """Periodic reorthogonalisation (reading Q28; the paper
    makes reorthogonalisation optional, and weighs its O(nK^2/2) cost,
    :260): Alg.1 with the full reorthogonalisation pass (l.12-18, O5) at the two
    consecutive iterations i = k p and k p + 1 (k = 1, 2, ...; Grcar's periodic scheme:
    reorthogonalising a single vector lets the three-term recurrence carry the lost
    orthogonality of its predecessor straight back); every other iteration is the plain
    three-term step. The same C iteration (orc_lanczos_iter) as O4, called with the
    per-iteration flag; period 1 is O4 with reorth, period > m is O4 without."""
    n = len(rowptr) - 1
    if v1vec is None:
        v1vec = v1(seed, n)
    rp, c, v = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    u = _c(v1vec, np.float64)
    V = np.zeros((m, n), np.float64)
    V[0] = u / np.sqrt(np.add.accumulate(u * u)[-1])  # sequential sum, as in oracle.c
    vt, vn = np.zeros(n), np.zeros(n)
    alpha, beta, ts = np.zeros(m), np.zeros(m + 1), np.zeros(1)
    mf, bd = m, False
    for i in range(1, m + 1):
        ro = 1 if (period >= 1 and (i % period == 0 or (i > 1 and (i - 1) % period == 0))) else 0
        if _load().orc_lanczos_iter(n, _p(rp), _p(c), _p(v), i, ro, tau, _p(V), _p(vt), _p(vn),
                                    _p(alpha), _p(beta), _p(ts)):
            mf, bd = i - 1, True
            break
    if not bd:
        beta[m] = np.sqrt(np.add.accumulate(vn * vn)[-1])
    lz = LanczosOut(alpha[:mf].copy(), beta[:mf + 1].copy(), V[:mf].copy(), mf, bd)
    theta, S, sw, conv = jacobi(tridiag_dense(lz.alpha, lz.beta))
    idx = select(theta, K)
    Y = ritz(lz.V, S, idx) if want_vectors else None
    rest = np.abs(lz.beta[mf] * S[mf - 1, idx]) if mf > 0 else np.zeros(0)
    return SolveOut(theta[idx], Y, theta, S, idx, lz, sw, conv, rest, extra={"period": period})


def solve_pro(rowptr, col, val, K: int, m: int, eps: float, seed: int = 1, v1vec=None,
              tau: float = 1e-12, want_vectors: bool = True) -> SolveOut:
    """Partial (selective) reorthogonalisation (reading Q29;
    Simon, Math. Comp. 42 (1984); the paper makes reorthogonalisation optional,
    PAPER.md:123). Every iteration is Alg.1's three-term step (O4 without reorth); the
    level of orthogonality of the new vector is estimated by Simon's recurrence
      beta_{j+1} w_{j+1,k} = beta_{k+1} w_{j,k+1} + (alpha_k - alpha_j) w_{j,k}
                             + beta_k w_{j,k-1} - beta_j w_{j-1,k} + theta_{j,k},
    theta_{j,k} = sign(.) eps (beta_{k+1} + beta_{j+1}) 0.3 (the deterministic worst case),
    w_{j+1,j} = psi = eps sqrt(n), w_{j,j} = 1, with beta_{j+1} the norm before any
    reorthogonalisation;
    when max_k |w_{j+1,k}| > sqrt(eps) the new vector is fully reorthogonalised (MGS
    against v_1..v_j, O5) and so is the next one, and the estimates of a
    reorthogonalised vector are reset to psi. eps = unit roundoff of the vector storage.
    extra["reorth_steps"] lists the reorthogonalised iterations."""
    n = len(rowptr) - 1
    if v1vec is None:
        v1vec = v1(seed, n)
    rp, c, v = _c(rowptr, np.int64), _c(col, np.int32), _c(val, np.float64)
    u = _c(v1vec, np.float64)
    V = np.zeros((m, n), np.float64)
    V[0] = u / np.sqrt(np.add.accumulate(u * u)[-1])
    vt, vn = np.zeros(n), np.zeros(n)
    alpha, beta, ts = np.zeros(m), np.zeros(m + 1), np.zeros(1)
    wp, wc = np.zeros(m + 2), np.zeros(m + 2)
    wc[1] = 1.0                      # w_{1,1}
    seps = np.sqrt(eps)
    mf, bd, force, steps = m, False, False, []
    for i in range(1, m + 1):
        if _load().orc_lanczos_iter(n, _p(rp), _p(c), _p(v), i, 0, tau, _p(V), _p(vt), _p(vn),
                                    _p(alpha), _p(beta), _p(ts)):
            mf, bd = i - 1, True
            break
        b = float(np.sqrt(np.add.accumulate(vn * vn)[-1]))   # beta_{i+1} before reorth
        ai, bi = alpha[i - 1], beta[i - 1]                    # alpha_i, beta_i
        new = np.zeros(m + 2)
        for k in range(1, i):
            t = beta[k] * wc[k + 1] + (alpha[k - 1] - ai) * wc[k]
            t = t + (beta[k - 1] * wc[k - 1] if k > 1 else 0.0)
            t = t - bi * wp[k]
            t = t + np.copysign(eps * (beta[k] + b) * 0.3, t)
            new[k] = t / b
        psi = eps * np.sqrt(n)
        new[i] = psi
        new[i + 1] = 1.0
        thr = i > 1 and float(np.max(np.abs(new[1:i]))) > seps
        if force or thr:
            for j in range(1, i + 1):                          # O5: MGS against v_1..v_i
                vj = V[j - 1]
                vn -= float(np.add.accumulate(vj * vn)[-1]) * vj
            new[1:i + 1] = psi
            steps.append(i)
        force = thr
        wp, wc = wc, new
    if not bd:
        beta[m] = np.sqrt(np.add.accumulate(vn * vn)[-1])
    lz = LanczosOut(alpha[:mf].copy(), beta[:mf + 1].copy(), V[:mf].copy(), mf, bd)
    theta, S, sw, conv = jacobi(tridiag_dense(lz.alpha, lz.beta))
    idx = select(theta, K)
    Y = ritz(lz.V, S, idx) if want_vectors else None
    rest = np.abs(lz.beta[mf] * S[mf - 1, idx]) if mf > 0 else np.zeros(0)
    return SolveOut(theta[idx], Y, theta, S, idx, lz, sw, conv, rest, extra={"reorth_steps": steps})
