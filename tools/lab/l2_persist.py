"""SpMV time on a large matrix (x > L2) with a persisting L2 window over the hub
prefix of x (TOPK_L2_PERSIST_MB), one process per setting is not needed: the window
is read at create."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synthgen as S
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
A = S.config_matrix(name)
import paper_2201_07498_b200 as T
for mb in (0, 16, 32, 64, 96):
    os.environ["TOPK_L2_PERSIST_MB"] = str(mb)
    with T.TopkEig(A, 16, "f32", "f64", m=16, profile=True, check_symmetry=False) as h:
        h.solve(seed=1, vectors=False)
        r = h.solve(seed=1, vectors=False)
        kt = h.kernel_times()
    print(json.dumps({"matrix": name, "persist_MB": mb, "spmv_ms_per_launch": round(kt["spmv"][0] / 16, 3),
                      "solve_ms": round(r.info["ms_solve"], 2), "top": r.eigenvalues[0]}), flush=True)
