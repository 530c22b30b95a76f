"""Cost of the two-pass SpMV (own-slot columns first) on one GPU:
G loopback parts with overlap = 1 (two passes) vs -1 (one pass), per-SpMV device time
summed over the parts (kernel_times class 'spmv' covers both passes of part 0; the
whole-solve time covers all parts). What the two passes cost here is what the overlap
must win back from the exchange when the parts are on different GPUs."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synthgen as S
import paper_2201_07498_b200 as T

wl = os.environ.get("OV_WL", "C3")
A = S.config_matrix(wl)
K = m = 16 if wl.startswith("C4") else 24
for G in (8,):
    for ov in (-1, 1):
        with T.TopkEig(A, K, "f32", "f64", m=m, parts=G, overlap=ov, profile=True, check_symmetry=False) as h:
            for i in range(3):
                r = h.solve(seed=1, vectors=False)
            kt = h.kernel_times()
        print(json.dumps({"workload": wl, "G": G, "overlap": ov, "part0_spmv_us_per_iter": round(kt["spmv"][0] / m * 1e3, 1),
                          "solve_ms_all_parts": round(r.info["ms_solve"], 3), "top": r.eigenvalues[0]}), flush=True)
