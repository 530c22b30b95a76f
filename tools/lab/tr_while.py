"""Thick restart on C3 (K = 24, m = 72, keep 36, tol 1e-5): device time per solve with
the WHILE-node graph vs unrolled cycles (restart_loop="unrolled"), for restart caps 10 and 40."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen as S, paper_2201_07498_b200 as T
A = S.config_matrix("C3")
for cond in (1, 0):
    for cap in (10, 40):
        with T.TopkEig(A, 24, "f32", "f64", m=72, restart_keep=36, max_restarts=cap, conv_tol=1e-5,
                       check_symmetry=False, restart_loop="auto" if cond else "unrolled") as h:
            ev = torch.zeros(24, dtype=torch.float64, device="cuda")
            h.solve_async(1, ev.data_ptr(), None); h.sync()
            st = torch.cuda.ExternalStream(h.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for i in range(5): h.solve_async(1, ev.data_ptr(), None)
            e1.record(st); h.sync()
            ms = e0.elapsed_time(e1) / 5
            r = h.solve(seed=1, vectors=True)
        print(json.dumps({"while_node": bool(cond), "cap": cap, "ms": round(ms, 3), "iterations": r.info["iterations"],
                          "restarts": r.info["restarts"], "stopped": r.info["converged_stop"],
                          "top": r.eigenvalues[0], "launches_captured": r.info["gpu_launches"]}), flush=True)
