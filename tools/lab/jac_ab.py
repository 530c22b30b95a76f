"""Jacobi (a12) device time per solve on C3S at m = 24 and 40 (single-CTA path), for A/B
of compile-time variants (tools/lab/variant_run.py)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synthgen as S
import paper_2201_07498_b200 as T
A = S.config_matrix("C3S")
for m in (24, 40):
    with T.TopkEig(A, 24, "f32", "f64", m=m, profile=True) as h:
        for i in range(3):
            r = h.solve(seed=1, vectors=False)
        kt = h.kernel_times()
    print(json.dumps({"m": m, "jacobi_ms": round(kt["jacobi"][0], 4), "sweeps": r.info["jacobi_sweeps"],
                      "top": r.eigenvalues[0]}), flush=True)
