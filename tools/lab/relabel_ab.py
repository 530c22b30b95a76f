"""Does the order of a big row's entries matter? C3 relabelled so that original ids
= degree-order positions (A' = P A P^T): then every row's canonical (ascending id)
order is ascending device column, i.e. big rows sorted by position. Per-launch SpMV
time of A and A' (same matrix up to the relabelling, same Krylov work)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import synthgen as S
import paper_2201_07498_b200 as T

A = S.config_matrix("C3")
n = A.n
deg = np.diff(A.rowptr)
order = np.lexsort((np.arange(n), -deg))        # position -> original row
pos = np.empty(n, np.int64); pos[order] = np.arange(n)
rows = np.repeat(np.arange(n), deg)
r2, c2 = pos[rows], pos[A.col]
key = r2 * n + c2
idx = np.argsort(key, kind="stable")
rp2 = np.zeros(n + 1, np.int64); np.add.at(rp2, r2 + 1, 1); rp2 = np.cumsum(rp2)
A2 = S.CSR(n, rp2, c2[idx].astype(np.int32), A.val[idx])
for name, M in (("canonical", A), ("sorted_by_position", A2), ("canonical", A), ("sorted_by_position", A2)):
    with T.TopkEig(M, 24, "f32", "f64", m=24, profile=True, check_symmetry=False) as h:
        for i in range(4):
            r = h.solve(seed=1, vectors=False)
        kt = h.kernel_times()
    print(json.dumps({"order": name, "spmv_us": round(kt["spmv"][0] / kt["spmv"][1] * 1e3, 1),
                      "solve_ms": round(r.info["ms_solve"], 3), "top": r.eigenvalues[0]}), flush=True)
