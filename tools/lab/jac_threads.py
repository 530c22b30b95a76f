"""Single-CTA Jacobi (m <= 40) time vs CTA size (TOPK_JAC_THREADS), C3S, m = 24 and 40."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synthgen as S, paper_2201_07498_b200 as T
A = S.config_matrix("C3S")
for m in (24, 40):
    for nt in (64, 96, 128, 192, 256, 384, 1024):
        os.environ["TOPK_JAC_THREADS"] = str(nt)
        with T.TopkEig(A, 24, "f32", "f64", m=m, profile=True) as h:
            for i in range(3): r = h.solve(seed=1, vectors=False)
            kt = h.kernel_times()
        print(json.dumps({"m": m, "threads": nt, "jacobi_ms": round(kt["jacobi"][0], 4), "top": r.eigenvalues[0]}), flush=True)
