"""Time-to-Top-K on C3 (FDF) for K = 8, 16, 24 (K in {8, 16, 24},
m in {K, 4K, 8K}): the bench's time_to_topk entries per K."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2201_07498_b200 as T
torch.cuda.set_device(0)
A = bench.make_matrix("C3")
for K in (8, 16, 24):
    wl = dict(bench.WORKLOADS["C3"], name="C3", K=K, m=K)
    kw = dict(storage="f32", compute="f64", device=0)
    out = bench.time_to_topk(T, A, wl, kw)
    print(json.dumps({"workload": "C3", "K": K, "time_to_topk": out}), flush=True)
