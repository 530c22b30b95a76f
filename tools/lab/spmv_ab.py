"""A/B of SpMV compile-time variants on C3 (FDF, K = m = 24): SpMV time per launch
and whole-solve time, one subprocess per library (TOPK_LIB). Variants are
built on the box by tools/build.py build_variant from the NAME=DEFINES list given on
the command line, e.g.  python tools/lab/spmv_ab.py nt768=TOPK_HUB_NT=768 gq4=TOPK_SPMV_GQ=4"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
CODE = r'''
import os, sys, json
sys.path.insert(0, %r)
import torch, synthgen as S, paper_2201_07498_b200 as T
if os.environ.get("AB_GRID"):  # nx,ny,drop: a weighted grid Laplacian instead of a named config
    nx, ny, dr = os.environ["AB_GRID"].split(",")
    A = S.grid_laplacian(int(nx), int(ny), float(dr), 6)
else:
    A = S.config_matrix(os.environ.get("AB_WL", "C3"))
with T.TopkEig(A, 24, "f32", "f64", m=24, profile=True, check_symmetry=False) as h:
    for i in range(3): h.solve(seed=1, vectors=False)
    kt = h.kernel_times()
with T.TopkEig(A, 24, "f32", "f64", m=24, check_symmetry=False) as h:
    ev = torch.zeros(24, dtype=torch.float64, device="cuda")
    Y = torch.zeros(24, A.n, dtype=torch.float32, device="cuda")
    for i in range(5): h.solve_async(1, ev.data_ptr(), Y.data_ptr(), "f32")
    h.sync()
    st = torch.cuda.ExternalStream(h.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(50): h.solve_async(1, ev.data_ptr(), Y.data_ptr(), "f32")
    e1.record(st); h.sync()
    ms = e0.elapsed_time(e1) / 50
    r = h.solve(seed=1, vectors=False)
print(json.dumps({"lib": os.environ.get("AB_NAME", "default"), "n": A.n, "nnz": A.nnz,
                  "matrix": os.environ.get("AB_GRID") or os.environ.get("AB_WL", "C3"),
                  "spmv_us": round(kt["spmv"][0] / 24 * 1e3, 1), "solve_ms": round(ms, 4),
                  "top": r.eigenvalues[0]}))
''' % ROOT


def main():
    from tools.build import build_variant
    libs = [("default", None)]
    os.makedirs(os.path.join(ROOT, "tools/lab/variants"), exist_ok=True)
    for spec in sys.argv[1:]:
        name, _, defs = spec.partition("=")
        out = os.path.join(ROOT, "tools/lab/variants", f"lib_{name}.so")
        from tools.build import deps
        if not (os.path.exists(out) and os.path.getmtime(out) > max(os.path.getmtime(f) for f in deps())):
            build_variant(out, [d for d in defs.split(",") if d])  # else prebuilt here (travels with gpurun)
        libs.append((name, out))
    for rep in range(2):
        for name, lib in libs:
            env = dict(os.environ, AB_NAME=name)
            if lib:
                env["TOPK_LIB"] = lib
            out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True, timeout=600)
            print(out.stdout.strip() or out.stderr[-800:], flush=True)


if __name__ == "__main__":
    main()
