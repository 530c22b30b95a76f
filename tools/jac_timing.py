#!/usr/bin/env python
"""Device time of the Jacobi solve (k_jacobi / k_jacobi_cl, one launch per solve)
against the Krylov dimension m, cluster path vs single-CTA global-memory path.
  python tools/jac_timing.py  -> one JSON line per (m, path)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthgen as S  # noqa: E402


def main():
    A = S.config_matrix("C3S")
    paths = {"single": dict(jacobi_path="single"),
             "cl8": dict(jacobi_path="cluster", jacobi_cluster=8),
             "cl16": dict(jacobi_path="cluster", jacobi_cluster=16),
             "default": {}}
    ms = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [24, 48, 64, 96, 130, 192, 256, 300]
    import paper_2201_07498_b200 as T
    for m in ms:
        for path, kw in paths.items():
            with T.TopkEig(A, 24, "f32", "f64", m=m, profile=True, **kw) as h:
                h.solve(seed=1, vectors=False)
                r = h.solve(seed=1, vectors=False)
                kt = h.kernel_times()
            print(json.dumps({"m": m, "path": path, "jacobi_ms": round(kt["jacobi"][0], 4),
                              "sweeps": r.info["jacobi_sweeps"], "solve_ms": round(r.info["ms_solve"], 3),
                              "top_eval": r.eigenvalues[0]}), flush=True)


if __name__ == "__main__":
    main()
