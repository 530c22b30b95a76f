#!/usr/bin/env python
"""bench.py — Lanczos iter/s (and SpMV HBM GB/s, time-to-Top-K) of the hot path.

Workload (default, BASELINE.json configs[2] "C3"): R-MAT power-law graph,
n = 4,194,304, nnz ~ 61M, FDF (f32 storage, f64 compute), K = m = 24. One
"step" = one full Top-K solve with the matrix resident in HBM: v1, 24 Lanczos
iterations (SpMV + alpha, fused recurrence + reorth multi-dot, correction +
beta), Jacobi on T, Ritz projection + normalisation.
value = Lanczos iterations per second of the whole job (m * steps / time).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  N > 1: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  (rows partitioned by nnz across ranks, NCCL allgather of v_i + scalars).

The reference arm (--impl reference) times the CPU oracle (oracle/, fp64,
single thread) on the same workload, one oracle Lanczos iteration per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_NOMINAL_GBS = 8000.0


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


WORKLOADS = {
    "C3": dict(desc="R-MAT S=22 (n=4,194,304), 31,457,280 samples, Graph500 (a,b,c)=(.57,.19,.19), "
                    "seed 22, symmetric, deduplicated, bf16-exact weights k/128",
               K=24, m=24, storage="f32", compute="f64"),
    "C3S": dict(desc="R-MAT S=16 (n=65,536), 491,520 samples, seed 16 (C3 shape, small)",
                K=24, m=24, storage="f32", compute="f64"),
    "C4": dict(desc="R-MAT ids over 2^27 (Graph500 a,b,c=.57,.19,.19) rejected if >= n, n=100,000,000, "
                    "1.41e9 samples, seed 27, symmetric, deduplicated, bf16-exact weights",
               K=16, m=16, storage="f32", compute="f64"),
    "C4X": dict(desc="R-MAT S=27 (n=2^27 = 134,217,728, GAP-kron's n, PAPER.md:180), 2.0e9 samples, seed 28, "
                     "symmetric, deduplicated -> nnz ~2.2e9 > 2^31 (64-bit offsets, SURVEY 8(f) NEXT-4)",
                K=16, m=16, storage="f32", compute="f64"),
    "C6": dict(desc="weighted Laplacian of a 4096 x 4096 4-neighbour grid, 25 % of edges dropped, seed 6, "
                    "row-major ids (n=16,777,216, nnz ~67M; mesh / road class of Table I, PAPER.md:167-177)",
               K=24, m=24, storage="f32", compute="f64"),
}


class ClockSampler:
    """nvidia-smi sampler running DURING the timed region (B200_PROFILING.md)."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(mx)) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_matrix(name: str):
    import synthgen as S
    return S.config_matrix(name)


def shared_matrix(name: str, rank: int, N: int, dist):
    """One process per GPU: rank 0 generates the matrix once and writes it to a file
    (synthgen.save_csr, /dev/shm when it has room, else /tmp); every rank maps it
    read-only, so the pages are shared and each rank's create reads only the row
    pointers and its own rows (plus its share of the symmetry hash). Returns
    (matrix, path or None); rank 0 removes the file at the end."""
    import shutil
    import synthgen as S
    if N == 1:
        return make_matrix(name), None
    tag = os.environ.get("TORCHELASTIC_RUN_ID", os.environ.get("MASTER_PORT", "0"))
    path = None
    if rank == 0:
        A = make_matrix(name)
        need = 8 * (A.n + 1) + 12 * A.nnz + 64
        d = "/dev/shm" if shutil.disk_usage("/dev/shm").free > 1.2 * need else "/tmp"
        path = os.path.join(d, f"topk_{name}_{tag}.csr")
        S.save_csr(path, A)
        del A
    obj = [path]
    dist.broadcast_object_list(obj, src=0)
    return S.load_csr_mmap(obj[0]), obj[0]


def gather_bound(nnz_g, t_ms):
    """The SpMV's other ceiling: one random 4/8-byte x gather
    per nonzero. profiles/gather_ceiling.json holds the measured B200 rate of
    uniform random gathers from an L2-resident vector (tools/lab/bwlab.cu)."""
    try:
        with open(os.path.join(ROOT, "profiles", "gather_ceiling.json")) as f:
            g = json.load(f)
        ach = nnz_g / (t_ms * 1e-3)
        return {"gathers_per_launch": int(nnz_g), "achieved_per_s": ach,
                "ceiling_per_s": g["gathers_per_s"], "frac": ach / g["gathers_per_s"], "source": g["source"]}
    except Exception:
        return None


def spmv_bytes(nnz_g, n_g, n_x, s, sv):
    """B_spmv = z_g (4 + s_v) + 4 (n_g + 1) + s n_x + s n_g."""
    return nnz_g * (4 + sv) + 4 * (n_g + 1) + s * n_x + s * n_g


def step_bytes(i, n_g, s):
    """B_step(i) = (2i + 4) n_g s (fused recurrence + multi-dot, then correction)."""
    return (2 * i + 4) * n_g * s


def cpu_baseline(A, wl):
    import oracle as O
    t0 = time.perf_counter()
    O.solve(A.rowptr, A.col, A.val, K=wl["K"], m=wl["m"], seed=1)
    dt = time.perf_counter() - t0
    return {"value": wl["m"] / dt, "unit": "iter/s", "cores": 1, "kind": "oracle",
            "seconds": dt,
            "sample": f"one full oracle solve of the same {wl['name']} matrix (v1 seed 1, m={wl['m']} "
                      "Lanczos iterations with MGS reorth, Jacobi, Ritz), single-threaded fp64 C",
            "host": host_info()}


def host_info():
    info = {"nproc": os.cpu_count()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["cpu"] = ln.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as f:
            info["mem_gb"] = round(int(f.readline().split()[1]) / 2 ** 20, 1)
    except Exception:
        pass
    return info


def run_reference(args, wl):
    """--impl reference: the CPU oracle on the same workload, rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    A = make_matrix(wl["name"])
    run = O.LanczosRun(A.rowptr, A.col, A.val, O.v1(1, A.n), wl["m"])
    for _ in range(args.warmup):
        run.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run.step()
    dt = time.perf_counter() - t0
    v = args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iter/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_of(wl, A, args.gpus),
            "cpu_baseline": {"value": v, "unit": "iter/s", "cores": 1, "kind": "oracle",
                             "sample": f"{args.steps} single oracle Lanczos iterations (SpMV + alpha + "
                                       f"recurrence + MGS reorth, Alg. 1) on the full {wl['name']} matrix, "
                                       f"cycling i = 1..{wl['m']}; Jacobi/Ritz excluded",
                             "host": host_info()},
            "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


METRIC = "lanczos_iter_per_s"


def config_of(wl, A, N):
    return {"workload": wl["name"], "matrix": wl["desc"], "n": int(A.n), "nnz": int(A.nnz),
            "K": wl["K"], "m": wl["m"],
            "precision": "FDF" if (wl["storage"], wl["compute"]) == ("f32", "f64") else
            f"{wl['storage']}-{wl['compute']}",
            "vector_storage": wl["storage"], "value_storage": wl["storage"], "compute": wl["compute"],
            "global_batch": 1, "parallelism": f"rows{N} (nnz-balanced row partition)",
            "l2": (f"inputs larger than L2: matrix {A.nnz * 8 / 1e9:.2f} GB (f32 values + int32 cols) + basis "
                   f"{(wl['m'] + 1) * A.n * 4 / 1e9:.2f} GB streamed per solve vs 126 MB L2; no flush needed"),
            "step": "one full Top-K solve (v1, m Lanczos iterations, Jacobi, Ritz) with M resident"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3", choices=list(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ttk", action="store_true", help="skip the time-to-Top-K m sweep")
    ap.add_argument("--sweep", action="store_true",
                    help="C5 precision sweep on the C3 matrix (report lines, not the bench line)")
    ap.add_argument("--exchange", default="allgather", choices=["allgather", "halo"],
                    help="vector exchange between ranks (N > 1): replicated allgather or halo (reading Q27)")
    ap.add_argument("--quality", action="store_true",
                    help="Fig. 3b analogue: eigenvector orthogonality and L2 error vs K, reorth on/off")
    args = ap.parse_args()
    if args.sweep:
        return run_sweep(args)
    if args.quality:
        return run_quality(args)
    wl = dict(WORKLOADS[args.workload], name=args.workload)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args, wl)

    ws, rank, local = dist_env()
    N = max(ws, 1)
    if N > 1 and rank > 0 and "OMP_NUM_THREADS" not in os.environ:
        # the host cores are shared by the ranks (rank 0 keeps all of them: it generates
        # the matrix while the others wait); set before libgomp loads
        os.environ["OMP_NUM_THREADS"] = str(max(1, (os.cpu_count() or N) // N))
    import torch
    if N != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {ws}", file=sys.stderr)
    torch.cuda.set_device(local)
    dist = None
    if N > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2201_07498_b200 as T

    A, shared_path = shared_matrix(wl["name"], rank, N, dist)
    nid = None
    if N > 1:
        obj = [T.nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    kw = dict(storage=wl["storage"], compute=wl["compute"], m=wl["m"], device=local)
    if N > 1:
        kw.update(parts=N, rank=rank, world=N, nccl_id=nid, exchange=args.exchange)
    # the headline value is timed without per-kernel event brackets (they add ~0.6 ms to
    # a C3 solve); the kernel breakdown and the roofline come from a second timed pass
    # on a handle that records them (profile=True), right after
    h = T.TopkEig(A, wl["K"], **kw)
    rp, _, _, npad = h.layout(0)
    n_g, nnz_g = len(rp) - 1, int(rp[-1])
    K, m = wl["K"], wl["m"]
    ev = torch.zeros(K, dtype=torch.float64, device="cuda")
    Y = torch.zeros(K, max(n_g, 1), dtype=torch.float32, device="cuda")
    stream = torch.cuda.ExternalStream(h.stream)

    for i in range(args.warmup):
        h.solve_async(1 + i, ev.data_ptr(), Y.data_ptr(), "f32")
        h.sync()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)  # let the sampler spin up before the timed region
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        h.solve_async(100 + i, ev.data_ptr(), Y.data_ptr(), "f32")
    e1.record(stream)
    info = h.sync()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = m * args.steps / (ms / 1e3)
    # per-solve device time for start vectors seeded 1..20 (median, p10, p90)
    per = []
    for sd in range(1, 21):
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        h.solve_async(sd, ev.data_ptr(), Y.data_ptr(), "f32")
        q1.record(stream)
        h.sync()
        per.append(q0.elapsed_time(q1))
    per_solve = {"seeds": "1..20", "median_ms": float(np.median(per)), "p10_ms": float(np.percentile(per, 10)),
                 "p90_ms": float(np.percentile(per, 90))}
    h.close()
    # kernel breakdown pass: same workload, CUDA events around every kernel of part 0
    # recorded inside the graph on the solve stream
    kwp = dict(kw)
    if N > 1:  # a fresh NCCL unique id per communicator
        obj = [T.nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        kwp["nccl_id"] = obj[0]
    hp = T.TopkEig(A, wl["K"], profile=True, **kwp)
    sp = torch.cuda.ExternalStream(hp.stream)
    for i in range(args.warmup):
        hp.solve_async(1 + i, ev.data_ptr(), Y.data_ptr(), "f32")
        hp.sync()
    nprof = max(1, min(args.steps, 20))
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(sp)
    for i in range(nprof):
        hp.solve_async(100 + i, ev.data_ptr(), Y.data_ptr(), "f32")
    p1.record(sp)
    hp.sync()
    prof_ms_step = p0.elapsed_time(p1) / nprof
    kt = hp.kernel_times()  # last solve of the breakdown pass
    hp.close()

    s = 4 if wl["storage"] == "f32" else 8 if wl["storage"] == "f64" else 2
    sv = s
    n_x = n_g if N == 1 else A.n
    b_spmv = spmv_bytes(nnz_g, n_g, n_x, s, sv)
    spmv_ms, spmv_n = kt["spmv"]
    t_spmv = spmv_ms / max(spmv_n, 1)
    spmv_gbs = b_spmv / (t_spmv * 1e-3) / 1e9
    peak, peak_src = load_peaks()
    b_step_tot = sum(step_bytes(i, n_g, s) for i in range(1, m + 1))
    stepcorr_ms = kt["step"][0] + kt["correct"][0]
    kernels = {c: {"ms_total": round(v[0], 4), "launches": v[1]} for c, v in kt.items()}
    kernels["spmv"]["gbs_algorithmic"] = round(spmv_gbs, 1)
    kernels["step+correct"] = {"ms_total": round(stepcorr_ms, 4),
                               "gbs_algorithmic": round(b_step_tot / (stepcorr_ms * 1e-3) / 1e9, 1)
                               if stepcorr_ms > 0 else None}

    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as f:
                d = json.load(f)
            if d.get("workload") == wl["name"] and d.get("n_gpus", 1) == N:
                traffic = d.get("spmv_dram_bytes_per_launch")
        except Exception:
            pass

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(T, A, wl, kw, args, N, rank, dist)

    ttk = None
    if N == 1 and not args.no_ttk:
        ttk = time_to_topk(T, A, wl, kw)

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu:
        cpu = cpu_baseline(A, wl)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": N, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(config_of(wl, A, N), **({"exchange": args.exchange} if N > 1 else {})),
                "time_to_topk_ms": ms_step,
                "time_to_topk": ttk,
                "spmv_hbm_gbs": spmv_gbs, "spmv_pct_of_8tbs": 100 * spmv_gbs / HBM_NOMINAL_GBS,
                "roofline": {"kernel": "k_spmv (SpMV + alpha partial, Alg.1 l.9-10)", "bound": "hbm",
                             "achieved": spmv_gbs, "peak": peak, "unit": "GB/s", "frac": spmv_gbs / peak,
                             "peak_source": peak_src, "traffic": traffic,
                             "algorithmic_bytes_per_launch": b_spmv, "avg_launch_ms": t_spmv,
                             "launches_timed": spmv_n,
                             "gather_bound": gather_bound(nnz_g, t_spmv)},
                "per_solve": per_solve,
                "kernels": kernels,
                "kernel_breakdown_pass": {"steps": nprof, "ms_per_step_with_events": round(prof_ms_step, 4),
                                          "note": "per-kernel CUDA events inside the graph (part 0); "
                                                  "the headline value is timed without them"},
                "cpu_baseline": cpu,
                "e2e": e2e,
                "gpu_launches": int(info["gpu_launches"]) * args.steps,
                "gpu_launches_per_step": int(info["gpu_launches"]),
                "clocks": clocks,
                "interconnect": None if N == 1 else {
                    "exchange": args.exchange, "overlap": "allgather on a second stream during the own-slot SpMV pass"
                    if args.exchange == "allgather" else "none (halo send/recv before the SpMV)",
                    "bytes_received_per_rank_per_solve": int(info["bytes_nvlink"]),
                    "bytes_per_iteration": int(info["bytes_nvlink"]) // max(1, m),
                    "gbs_if_spread_over_lanczos_phase": round(info["bytes_nvlink"] / max(info["ms_lanczos"], 1e-9) / 1e6, 1),
                    "nvlink5_gbs_per_direction": 900,
                    "frac_of_nvlink5": round(info["bytes_nvlink"] / max(info["ms_lanczos"], 1e-9) / 1e6 / 900, 4),
                    "note": "modelled bytes (topk_eig_info_t.bytes_nvlink); the exchange is not timed separately"},
                "solve_info": {k: info[k] for k in ("k_found", "iterations", "breakdown", "jacobi_sweeps",
                                                    "jacobi_converged")},
                "paper_context": "paper (V100, fp32): 67x vs 104-thread ARPACK, 1.9x vs Alveo U280 FPGA "
                                 "(PAPER.md:21,219); context only, not comparable"}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        if rank == 0 and shared_path:
            os.remove(shared_path)
        dist.destroy_process_group()
    return 0


def time_to_topk(T, A, wl, kw, reps=5):
    """SURVEY 8(d) time-to-Top-K: device time of one solve (matrix resident) at
    Krylov dimension m in {K, 2K, 4K, 8K}, and how many of the K Ritz pairs are
    converged by the residual estimate |beta_{m+1} s_{m,k}| <= 1e-5 |theta_1|
    (reading Q6; equal to the true residual to ~1e-15)."""
    import torch
    K = wl["K"]
    out = {}
    for f in (1, 2, 4, 8):
        m = f * K
        kw2 = dict(kw, m=m)
        with T.TopkEig(A, K, check_symmetry=False, **kw2) as h:
            ev = torch.zeros(K, dtype=torch.float64, device="cuda")
            h.solve_async(1, ev.data_ptr(), None)
            h.sync()
            stream = torch.cuda.ExternalStream(h.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(reps):
                h.solve_async(2 + i, ev.data_ptr(), None)
            e1.record(stream)
            h.sync()
            ms = e0.elapsed_time(e1) / reps
            r = h.solve(seed=1, vectors=False)
        conv = int(np.sum(r.residual_est <= 1e-5 * abs(r.eigenvalues[0])))
        out[f"m={m}"] = {"ms": round(ms, 3), "converged_of_K": conv}
    # convergence-driven stop (reading Q25): m <= 8K, checked every c iterations
    for c in (8, K):
        with T.TopkEig(A, K, check_symmetry=False, conv_tol=1e-5, conv_check=c, **dict(kw, m=8 * K)) as h:
            ev = torch.zeros(K, dtype=torch.float64, device="cuda")
            h.solve_async(1, ev.data_ptr(), None)
            h.sync()
            stream = torch.cuda.ExternalStream(h.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(reps):
                h.solve_async(1, ev.data_ptr(), None)
            e1.record(stream)
            h.sync()
            ms = e0.elapsed_time(e1) / reps
            r = h.solve(seed=1, vectors=False)
        conv = int(np.sum(r.residual_est <= 1e-5 * abs(r.eigenvalues[0])))
        out[f"adaptive tol=1e-5 c={c}"] = {"ms": round(ms, 3), "iterations": r.info["iterations"],
                                           "converged_of_K": conv, "stopped": bool(r.info["converged_stop"])}
    # partial reorthogonalisation (reading Q29) at m = 8K
    with T.TopkEig(A, K, check_symmetry=False, reorth=3, **dict(kw, m=8 * K)) as h:
        ev = torch.zeros(K, dtype=torch.float64, device="cuda")
        h.solve_async(1, ev.data_ptr(), None)
        h.sync()
        stream = torch.cuda.ExternalStream(h.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(reps):
            h.solve_async(1, ev.data_ptr(), None)
        e1.record(stream)
        h.sync()
        ms = e0.elapsed_time(e1) / reps
        r = h.solve(seed=1, vectors=False)
    conv = int(np.sum(r.residual_est <= 1e-5 * abs(r.eigenvalues[0])))
    out[f"partial reorth m={8 * K}"] = {"ms": round(ms, 3), "reorth_passes": r.info["reorth_passes"],
                                        "converged_of_K": conv}
    # thick restart (reading Q26): basis of m = 3K (2K+1 .. 3K steps per cycle), stop at tol;
    # the restart cycles run in a CUDA-graph WHILE node, so the cap costs nothing
    for mr, keep in ((3 * K, 3 * K // 2), (4 * K, 2 * K)):
        with T.TopkEig(A, K, check_symmetry=False, conv_tol=1e-5, restart_keep=keep, max_restarts=40,
                       **dict(kw, m=mr)) as h:
            ev = torch.zeros(K, dtype=torch.float64, device="cuda")
            h.solve_async(1, ev.data_ptr(), None)
            h.sync()
            stream = torch.cuda.ExternalStream(h.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(reps):
                h.solve_async(1, ev.data_ptr(), None)
            e1.record(stream)
            h.sync()
            ms = e0.elapsed_time(e1) / reps
            r = h.solve(seed=1, vectors=False)
        conv = int(np.sum(r.residual_est <= 1e-5 * abs(r.eigenvalues[0])))
        out[f"thick restart m={mr} keep={keep} tol=1e-5"] = {
            "ms": round(ms, 3), "iterations": r.info["iterations"], "restarts": r.info["restarts"],
            "converged_of_K": conv, "stopped": bool(r.info["converged_stop"])}
    return out


def run_e2e(T, A, wl, kw, args, N, rank, dist):
    """Same metric through the public API with host buffers: every step creates
    the solver from the host CSR (H2D upload inside), solves, and copies the
    eigenpairs back to host memory (D2H)."""
    import torch
    steps = max(1, min(args.e2e_steps, args.steps))
    times = []
    h2d = d2h = 0
    for i in range(steps + 1):
        kwi = dict(kw)
        if dist:
            # a fresh NCCL unique id per communicator (ids are not reusable)
            obj = [T.nccl_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            kwi["nccl_id"] = obj[0]
            dist.barrier()
        t0 = time.perf_counter()
        with T.TopkEig(A, wl["K"], **kwi) as h2:  # default create: symmetry check on
            r = h2.solve(seed=500 + i, vectors=True, vec_dtype="f32")
            rp, _, _, _ = h2.layout(0) if i == 0 else (None, None, None, None)
            if i == 0:
                n_g, z_g = len(rp) - 1, int(rp[-1])
                s = 4 if wl["storage"] == "f32" else 8
                # create uploads the canonical CSR slice (two int64 row pointers: the input
                # one and the degree-ordered one, int32 columns, values in the storage dtype),
                # the column map (int32 per column), perm + inverse (int32 per row) and the
                # chunk / SELL / item tables; the device builds the SpMV layout from them
                h2d = 16 * (n_g + 1) + z_g * (4 + s) + 4 * A.n + 8 * n_g + 24 * (z_g // 8192 + 1) \
                    + 16 * (n_g // 32 + 1) + 64
                d2h = 8 * wl["K"] * 2 + 4 * wl["K"] * A.n
        dt = time.perf_counter() - t0
        if i > 0:  # first call warms the process (cudaMalloc pools, module load)
            times.append(dt)
    t = max(times)
    if dist:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    return {"value": wl["m"] / float(np.mean(times)) if not dist else wl["m"] / t, "unit": "iter/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "s_per_step": float(np.mean(times)),
            "note": "create with the default options (host canonicalise + symmetry check + partition + layout "
                    "tables, CSR H2D through pinned staging, device-side layout scatter) + solve + eigenvalues/eigenvectors "
                    "(f32) D2H through pinned staging, wall clock; first call untimed (module load, memory pools)"}


SWEEP_ARMS = [  # (name, vector storage, compute, value storage)
    ("DDD", "f64", "f64", "f64"),
    ("FDF", "f32", "f64", "f32"),
    ("FFF", "f32", "f32", "f32"),
    ("bf16val-f32vec-f64", "f32", "f64", "bf16"),
    ("bf16val-bf16vec-f64", "bf16", "f64", "bf16"),
]


def run_sweep(args):
    """C5 (BASELINE.json configs[4]; the paper's Fig. 4 analogue):
    accuracy vs time of every (storage, compute) arm on the C3 matrix, K = 24,
    m in {24, 192}. Accuracy is normwise against the DDD arm (itself checked
    against the fp64 oracle by the parity tests); bf16 vectors are report-only
    (reading Q21). One JSON line per (arm, m)."""
    import torch
    import paper_2201_07498_b200 as T
    torch.cuda.set_device(0)
    A = make_matrix("C3")
    K = 24
    for m in (24, 192):
        ref = None
        for name, st, ct, vs in SWEEP_ARMS:
            with T.TopkEig(A, K, storage=st, compute=ct, values_storage=vs, m=m, check_symmetry=False) as h:
                ev = torch.zeros(K, dtype=torch.float64, device="cuda")
                for i in range(args.warmup):
                    h.solve_async(1, ev.data_ptr(), None)
                    h.sync()
                stream = torch.cuda.ExternalStream(h.stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = max(3, min(args.steps, 20))
                e0.record(stream)
                for i in range(reps):
                    h.solve_async(1, ev.data_ptr(), None)
                e1.record(stream)
                h.sync()
                ms = e0.elapsed_time(e1) / reps
                r = h.solve(seed=1, vectors=False)
                _, _, theta = h.tridiag()
            theta = np.sort(theta)
            if ref is None:
                ref = (theta, r.eigenvalues)
            errn = float(np.abs(theta - ref[0]).max() / np.abs(ref[0]).max()) if len(theta) == len(ref[0]) else None
            top = float(np.nanmax(np.abs(r.eigenvalues - ref[1])) / abs(ref[1][0]))
            print(json.dumps({"kind": "precision_sweep", "workload": "C5 (C3 matrix)", "arm": name, "K": K, "m": m,
                              "ms_per_solve": ms, "iter_per_s": m / (ms / 1e3),
                              "ritz_normwise_err_vs_DDD": errn, "topK_err_vs_DDD": top,
                              "residual_est_max_rel": float(np.nanmax(r.residual_est) / abs(r.eigenvalues[0])),
                              "report_only": vs == "bf16" and st == "bf16"}), flush=True)
    return 0


def eigen_quality(A, Y, theta):
    """Fig. 3b metrics of K returned eigenpairs against the fp64
    matrix: the mean angle between every pair of eigenvectors (arccos |y_j . y_k|,
    90 degrees for exact ones) and the mean L2 reconstruction error ||M y - lambda y||
    (y unit norm, unnormalised by ||M||, as the paper plots it)."""
    import scipy.sparse as sp
    M = sp.csr_matrix((A.val, A.col, A.rowptr), shape=(A.n, A.n))
    Y = np.asarray(Y, np.float64)
    Y = Y / np.linalg.norm(Y, axis=1, keepdims=True)
    G = np.abs(Y @ Y.T)
    iu = np.triu_indices(len(Y), 1)
    ang = np.degrees(np.arccos(np.clip(G[iu], 0.0, 1.0)))
    R = (M @ Y.T).T - theta[:, None] * Y
    res = np.linalg.norm(R, axis=1)
    return {"mean_angle_deg": float(ang.mean()) if len(ang) else None,
            "min_angle_deg": float(ang.min()) if len(ang) else None,
            "max_abs_dot": float(G[iu].max()) if len(ang) else None,
            "mean_l2_err": float(res.mean()), "max_l2_err": float(res.max()),
            "residuals": res}


def run_quality(args):
    """NEXT-3: the paper's Fig. 3b on the C3 matrix -- for K = 8, 16, 24
    at m = K, reorthogonalisation on (CGS) and off, in DDD, FDF and
    FFF: mean pairwise eigenvector angle and mean ||M y - lambda y||; plus how well the
    device residual estimate |beta_{m+1} s_{m,k}| tracks the measured residual. One JSON
    line per (arm, reorth, K); report lines, not the bench line."""
    import torch
    import paper_2201_07498_b200 as T
    torch.cuda.set_device(0)
    A = make_matrix("C3")
    arms = [a for a in SWEEP_ARMS if a[0] in ("DDD", "FDF", "FFF")]
    for name, st, ct, vs in arms:
        for reorth, period in ((1, 1), (1, 4), (3, 1), (-1, 1)):
            for K in (8, 16, 24):
                with T.TopkEig(A, K, storage=st, compute=ct, values_storage=vs, m=K, reorth=reorth,
                               reorth_period=period, check_symmetry=False) as h:
                    r = h.solve(seed=1, vectors=True, vec_dtype="f64")
                kf = len(r.eigenvectors)
                q = eigen_quality(A, r.eigenvectors, r.eigenvalues[:kf])
                est = np.asarray(r.residual_est[:kf])
                res = q.pop("residuals")
                gap = float(np.max(np.abs(est - res)) / abs(r.eigenvalues[0]))
                print(json.dumps({"kind": "quality", "workload": "C3", "arm": name,
                                  "reorth": {1: "cgs" if period == 1 else f"cgs pairs every {period}", 3: "partial (Simon)",
                                             -1: "off"}[reorth], "reorth_passes": r.info["reorth_passes"],
                                  "K": K, "m": K, "k_found": kf,
                                  **q, "residual_est_vs_measured_max_rel": gap}), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
