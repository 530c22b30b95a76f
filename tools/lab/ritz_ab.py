"""A/B of the Ritz output pass (a14) on C3 (FDF, K = m = 24, f32 vectors): fp64
tensor-core k_ritz_mma vs the CUDA-core k_ritz, per-kernel event times and the
eigenvector difference between the two paths."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import synthgen as S
import paper_2201_07498_b200 as T

A = S.config_matrix(os.environ.get("AB_WL", "C3"))
res = {}
for path in ("auto", "cuda_cores", "auto"):
    with T.TopkEig(A, 24, "f32", "f64", m=24, profile=True, check_symmetry=False, ritz_path=path) as h:
        for i in range(3):
            r = h.solve(seed=1, vectors=True, vec_dtype="f32")
        kt = h.kernel_times()
    res[path] = r.eigenvectors.astype(np.float64)
    print(json.dumps({"ritz_path": path, "ritz_out_ms": round(kt["ritz_out"][0], 4),
                      "unperm_ms": round(kt["unperm"][0], 4), "solve_ms": round(r.info["ms_solve"], 3),
                      "ms_ritz_phase": round(r.info["ms_ritz"], 4)}), flush=True)
d = max(min(np.linalg.norm(a - b), np.linalg.norm(a + b)) for a, b in zip(res["auto"], res["cuda_cores"]))
print(json.dumps({"max_vector_diff": float(d)}))
