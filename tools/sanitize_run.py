"""Small solves through the C ABI for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): C1 (COO input, duplicates), a star matrix whose rows sit at
the SpMV layout boundaries (127/128/129 SELL vs big row, 8191/8192/8193/16385 one vs
several chunks finished by the last-arriving one), C3S in FDF with G = 3 loopback
parts, eager launches (the sanitizer follows graph launches too, eager is clearer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synthgen as S
import oracle as O
import paper_2201_07498_b200 as T

c = S.config_matrix("C1")
rp, col, val = O.coo_to_csr(c.n, c.row, c.col, c.val)
cases = [("C1", S.CSR(c.n, rp, col, val), "f64", 1, 16),
         ("stars", S.stars([8191, 8192, 8193, 16385], dense=[127, 128, 129, 3]), "f64", 1, 24),
         ("stars G3", S.stars([8191, 8192, 8193, 16385], dense=[127, 128, 129, 3]), "f32", 3, 24),
         ("C3S G3", S.config_matrix("C3S"), "f32", 3, 24)]
graph = os.environ.get("SAN_GRAPH", "0") == "1"
for name, A, st, G, m in cases:
    with T.TopkEig(A, 8, st, "f64", m=m, parts=G, use_graph=graph) as h:
        r = h.solve(seed=1)
        y = h.debug_spmv(np.linspace(-1, 1, A.n))
    print(name, "ok", r.info["k_found"], float(r.eigenvalues[0]), float(np.abs(y).max()), flush=True)
