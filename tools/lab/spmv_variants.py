"""A/B of SpMV compile-time variants (tools/build.py build_variant) on C3: per-launch
SpMV time and whole-solve time, one subprocess per library (TOPK_LIB)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = r'''
import os, sys, json
sys.path.insert(0, %r)
import torch, synthgen as S, paper_2201_07498_b200 as T
A = S.config_matrix("C3")
with T.TopkEig(A, 24, "f32", "f64", m=24, profile=True, check_symmetry=False) as h:
    for i in range(3): h.solve(seed=1, vectors=True, vec_dtype="f32")
    kt = h.kernel_times()
with T.TopkEig(A, 24, "f32", "f64", m=24, check_symmetry=False) as h:
    ev = torch.zeros(24, dtype=torch.float64, device="cuda")
    Y = torch.zeros(24, A.n, dtype=torch.float32, device="cuda")
    for i in range(5): h.solve_async(1, ev.data_ptr(), Y.data_ptr(), "f32")
    h.sync()
    st = torch.cuda.ExternalStream(h.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(100): h.solve_async(1, ev.data_ptr(), Y.data_ptr(), "f32")
    e1.record(st); h.sync()
    ms = e0.elapsed_time(e1) / 100
print(json.dumps({"lib": os.environ.get("TOPK_LIB", "default"), "spmv_us": round(kt["spmv"][0] / 24 * 1e3, 1), "ritz_ms": round(kt["ritz_out"][0], 4), "unperm_ms": round(kt["unperm"][0], 4), "solve_ms": round(ms, 4)}))
''' % ROOT
libs = [None] + sorted(os.path.join(ROOT, "tools/lab/variants", f) for f in os.listdir(os.path.join(ROOT, "tools/lab/variants")) if f.endswith(".so"))
for rep in range(2):
    for lib in libs:
        env = dict(os.environ)
        if lib:
            env["TOPK_LIB"] = lib
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
        print(out.stdout.strip() or out.stderr[-500:], flush=True)
