"""Thick-restart diagnostics on C3S (DDD): basis orthogonality and explicit
residuals vs estimates after R restarts, GPU vs oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, scipy.sparse as sp
import synthgen as S, oracle as O, paper_2201_07498_b200 as T
A = S.config_matrix("C3S")
M = sp.csr_matrix((A.val, A.col, A.rowptr), shape=(A.n, A.n))
K, m, keep = 16, 48, 24
for R in (0, 1, 2, 4):
    with T.TopkEig(A, K, "f64", "f64", m=m, restart_keep=keep, max_restarts=R) as h:
        r = h.solve(seed=5)
        V = h.basis()
    ref = O.solve_thick_restart(A.rowptr, A.col, A.val, K, m, keep, R, seed=5)
    orth = np.abs(V @ V.T - np.eye(len(V))).max()
    orth_o = np.abs(ref.lanczos.V @ ref.lanczos.V.T - np.eye(m)).max()
    res = [np.linalg.norm(M @ y - t * y) for y, t in zip(r.eigenvectors, r.eigenvalues)]
    reso = [np.linalg.norm(M @ y - t * y) for y, t in zip(ref.eigenvectors, ref.eigenvalues)]
    print(f"R={R} gpu orth {orth:.2e} oracle orth {orth_o:.2e} | max|res-est| gpu {np.max(np.abs(np.array(res)-r.residual_est)):.2e} "
          f"oracle {np.max(np.abs(np.array(reso)-ref.residual_est)):.2e} | iters {r.info['iterations']}", flush=True)
    if R == 1:
        # column-wise orthogonality profile
        G = np.abs(V @ V.T - np.eye(len(V)))
        print("  worst column pairs", [tuple(x) for x in np.argwhere(G > 1e-10)[:10]])
