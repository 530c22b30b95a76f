"""topk_eig_create stage times on C3 (TOPK_TRACE=1), three creates in one process."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["TOPK_TRACE"] = "1"
import numpy as np
import synthgen as S, paper_2201_07498_b200 as T
A = S.config_matrix(sys.argv[1] if len(sys.argv) > 1 else "C3")
for rep in range(int(os.environ.get("REPS", "5"))):
    t0 = time.perf_counter()
    h = T.TopkEig(A, 24, "f32", "f64")  # default options (symmetry check on)
    t1 = time.perf_counter()
    r = h.solve(seed=1, vectors=True, vec_dtype="f32")
    t2 = time.perf_counter()
    h.close()
    t3 = time.perf_counter()
    print(f"rep {rep}: create {t1 - t0:.3f} s, solve+D2H {t2 - t1:.3f} s, destroy {t3 - t2:.3f} s", flush=True)
