"""Achieved bandwidth of the reorthogonalisation kernels (k_stepw passes, k_correct)
over a whole solve at Krylov dimension m on C3 (FDF), from the per-class device times."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synthgen as S, paper_2201_07498_b200 as T
A = S.config_matrix("C3")
for m in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "24,96,192").split(",")]:
    with T.TopkEig(A, 24, "f32", "f64", m=m, profile=True, check_symmetry=False) as h:
        h.solve(seed=1, vectors=False)
        h.solve(seed=1, vectors=False)
        kt = h.kernel_times()
        npad = h.layout(0)[3]
    s = 4
    col = npad * s
    step_b = corr_b = 0
    for i in range(1, m + 1):
        npass = 1 if i <= 17 else (i + 15) // 16
        step_b += (i + 4 + 2 * (npass - 1)) * col   # V[0..i) + y + u_i + u_{i-1} + w write, w re-read/written per extra pass
        corr_b += (i + 2) * col
    st, co = kt["step"][0], kt["correct"][0]
    print(json.dumps({"m": m, "step_ms": round(st, 3), "step_TBps": round(step_b / st / 1e9, 2),
                      "correct_ms": round(co, 3), "correct_TBps": round(corr_b / co / 1e9, 2),
                      "spmv_ms": round(kt["spmv"][0], 3), "jacobi_ms": round(kt["jacobi"][0], 3)}), flush=True)
