"""A/B: exact-width correction (k_correctw) vs 8-column batches (k_correct) on C3."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import os, sys, json
sys.path.insert(0, %r)
import torch, synthgen as S, paper_2201_07498_b200 as T
A = S.config_matrix("C3")
with T.TopkEig(A, 24, "f32", "f64", m=24, profile=True, check_symmetry=False) as h:
    for i in range(3): h.solve(seed=1, vectors=False)
    kt = h.kernel_times()
with T.TopkEig(A, 24, "f32", "f64", m=24, check_symmetry=False) as h:
    ev = torch.zeros(24, dtype=torch.float64, device="cuda")
    for i in range(5): h.solve_async(1, ev.data_ptr(), None)
    h.sync()
    st = torch.cuda.ExternalStream(h.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(100): h.solve_async(1, ev.data_ptr(), None)
    e1.record(st); h.sync()
    ms = e0.elapsed_time(e1) / 100
    r = h.solve(seed=1, vectors=False)
print(json.dumps({"corrw": os.environ.get("TOPK_NO_CORRW", "0") != "1", "correct_ms": round(kt["correct"][0], 4),
                  "step_ms": round(kt["step"][0], 4), "solve_ms": round(ms, 4), "top": r.eigenvalues[0]}))
''' % ROOT
for rep in range(2):
    for off in ("0", "1"):
        env = dict(os.environ, TOPK_NO_CORRW=off)
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
        print(out.stdout.strip() or out.stderr[-400:], flush=True)
