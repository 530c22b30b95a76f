"""Loopback G-part solve of a large matrix with the replicated-vector exchange vs the
halo exchange (reading Q27): part 0's SpMV time per launch (profile brackets part 0),
whole-solve device time, and the exchange volume per iteration."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import synthgen as S, paper_2201_07498_b200 as T
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
G = int(sys.argv[2]) if len(sys.argv) > 2 else 8
A = S.config_matrix(name)
nh = [T.plan_halo(A, G, g)["n_halo"] for g in range(G)] if A.n <= 10_000_000 else None
for ex in ("allgather", "halo"):
    with T.TopkEig(A, 16, "f32", "f64", m=16, parts=G, exchange=ex, profile=True, check_symmetry=False) as h:
        h.solve(seed=1, vectors=False)
        r = h.solve(seed=1, vectors=False)
        kt = h.kernel_times()
    print(json.dumps({"matrix": name, "G": G, "exchange": ex, "part0_spmv_ms_per_launch": round(kt["spmv"][0] / 16, 3),
                      "solve_ms": round(r.info["ms_solve"], 2), "top": r.eigenvalues[0],
                      "halo_entries_per_part": nh}), flush=True)
