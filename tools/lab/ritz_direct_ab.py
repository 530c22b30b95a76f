"""Ritz output pass: position order + un-permute vs the direct row-order pass
(k_ritz_mma DIRECT) on C3 / C6 (FDF, K = m = 24): kernel times per solve and
whether both give the same eigenvectors bit for bit. The direct variant and its
ritz_path values ("tc_unpermute", "tc_direct") were removed after this measurement
(slower, profiles/r02_ritz_direct_ab.jsonl); the script documents the run."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import synthgen as S
import paper_2201_07498_b200 as T

for name in sys.argv[1:] or ["C3", "C6"]:
    A = S.config_matrix(name)
    Y = {}
    for path in ("tc_unpermute", "tc_direct", "auto"):
        with T.TopkEig(A, 24, "f32", "f64", m=24, profile=True, check_symmetry=False, ritz_path=path) as h:
            for i in range(3):
                r = h.solve(seed=1, vectors=True, vec_dtype="f32")
            kt = h.kernel_times()
        Y[path] = r.eigenvectors
        print(json.dumps({"matrix": name, "ritz_path": path, "ritz_ms": round(kt["ritz_out"][0], 4),
                          "unperm_ms": round(kt["unperm"][0], 4), "unperm_launches": kt["unperm"][1],
                          "solve_ms": round(r.info["ms_solve"], 3)}), flush=True)
    print(json.dumps({"matrix": name, "direct_equals_unpermute_bitwise": bool(np.array_equal(Y["tc_direct"], Y["tc_unpermute"]))}))
