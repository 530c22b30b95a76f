"""A/B: per-solve device time on C3 with/without programmatic dependent launch
and with/without the per-kernel profiling events (bench's kernel breakdown)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import synthgen as S
A = S.config_matrix("C3")
import paper_2201_07498_b200 as T
torch.cuda.set_device(0)
res = {}
for rep in range(2):
    for pdl in (0, 1):
        for prof in (False, True):
            os.environ["TOPK_NO_PDL"] = "0" if pdl else "1"
            with T.TopkEig(A, 24, "f32", "f64", m=24, profile=prof, check_symmetry=False) as h:
                ev = torch.zeros(24, dtype=torch.float64, device="cuda")
                for i in range(5):
                    h.solve_async(1, ev.data_ptr(), None)
                h.sync()
                st = torch.cuda.ExternalStream(h.stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for i in range(100):
                    h.solve_async(1, ev.data_ptr(), None)
                e1.record(st)
                h.sync()
                ms = e0.elapsed_time(e1) / 100
            res.setdefault((pdl, prof), []).append(ms)
for (pdl, prof), v in sorted(res.items()):
    print(json.dumps({"pdl": pdl, "profile_events": prof, "ms_per_solve": [round(x, 4) for x in v]}))
