"""Host-side logic of the N > 1 path on CPU: two processes (torch.distributed,
gloo, world_size 2) each plan their own part through the host-only C ABI
(topk_eig_plan_partition / topk_eig_plan_layout), exactly what a rank does in
topk_eig_create, and run the paper's per-iteration exchange protocol
(replicated v_i, alpha / beta partial sums) with numpy on
their layout. Checks: every rank derives the same boundaries; the parts'
layouts equal the oracle's; the padded-slot allgather + remapped columns give
the global SpMV; alpha and ||w||^2 summed from rank-ordered partials agree on
both ranks bitwise and with the single-part value to rounding."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synthgen as S

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2201_07498_b200 as T
        A = S.rmat(12, 40_000, 12)
        G = WORLD
        b = T.plan_partition(A.rowptr, G)
        allb = [torch.zeros(G + 1, dtype=torch.int64) for _ in range(G)]
        dist.all_gather(allb, torch.from_numpy(b))
        same_b = all(np.array_equal(x.numpy(), b) for x in allb)
        L = T.plan_layout(A, G, rank, "f64")
        rp, col, val, npad, perm = L["rowptr"], L["col"], L["val"], L["n_pad"], L["perm"]
        orp, ocol, oval, onpad, operm = O.layout(A.rowptr, A.col, A.val, G, O.partition(A.rowptr, G), rank,
                                                 "f64", with_perm=True)
        layout_ok = (np.array_equal(rp, orp) and np.array_equal(col, ocol) and np.array_equal(val, oval)
                     and npad == onpad and np.array_equal(perm, operm))
        # replicated v_i: each rank publishes its padded slot
        v = O.v1(7, A.n)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        slot = np.zeros(npad)
        slot[: r1 - r0] = v[r0 + perm]  # part vectors live in hub-first position order
        slots = [torch.zeros(npad, dtype=torch.float64) for _ in range(G)]
        dist.all_gather(slots, torch.from_numpy(slot))
        replica = torch.cat(slots).numpy()
        # local SpMV on the remapped columns, then the alpha partial (Alg.1 l.9-10)
        xg = replica[col]
        y = np.array([np.dot(val[rp[r]:rp[r + 1]], xg[rp[r]:rp[r + 1]]) for r in range(r1 - r0)])
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(G)]
        vloc = v[r0 + perm]
        dist.all_gather(parts, torch.tensor([np.dot(y, vloc)], dtype=torch.float64))
        alpha = 0.0
        for p in parts:  # rank order (reading Q16)
            alpha += float(p[0])
        w = y - alpha * vloc
        nparts = [torch.zeros(1, dtype=torch.float64) for _ in range(G)]
        dist.all_gather(nparts, torch.tensor([np.dot(w, w)], dtype=torch.float64))
        wn = 0.0
        for p in nparts:
            wn += float(p[0])
        yg = O.spmv(A.rowptr, A.col, A.val, v)
        q.put((rank, same_b, layout_ok, y, alpha, wn, float(np.dot(yg, v)), yg[r0 + perm]))
    finally:
        dist.destroy_process_group()


def test_two_rank_plan_and_exchange_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    for rank, same_b, layout_ok, y, alpha, wn, alpha_g, yg in out:
        assert same_b, "ranks derived different partitions"
        assert layout_ok, f"rank {rank} layout differs from the oracle's"
        assert np.abs(y - yg).max() <= 1e-12 * max(1.0, np.abs(yg).max())
        assert abs(alpha - alpha_g) <= 1e-12 * max(1.0, abs(alpha_g))
    # scalars identical on every rank (rank-ordered sums of the same partials)
    assert out[0][4] == out[1][4] and out[0][5] == out[1][5]


def _halo_worker(rank, port, q):
    """Halo exchange (reading Q27) on two gloo ranks: each rank plans its halo
    (topk_eig_plan_halo), sends its request lists to the owners, answers the
    requests it receives from its own slot, and runs its SpMV on the compact vector
    [own slot | received entries] -- the protocol topk_eig_create / exch_halo run
    with NCCL send/recv -- against the full SpMV."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2201_07498_b200 as T
        A = S.rmat(12, 40_000, 13)
        G = WORLD
        b = T.plan_partition(A.rowptr, G)
        L = T.plan_layout(A, G, rank, "f64")
        H = T.plan_halo(A, G, rank)
        rp, col, val, npad, perm = L["rowptr"], L["col"], L["val"], L["n_pad"], L["perm"]
        off, hpos = H["off"], H["pos"]
        # request lists to the owners (what NCCL send/recv carries once at create)
        reqs = [None] * G
        dist.all_gather_object(reqs, {qq: hpos[off[qq]:off[qq + 1]].tolist() for qq in range(G) if qq != rank})
        # the iteration: own slot, answer each peer's requests, receive mine
        v = O.v1(9, A.n)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        own = np.zeros(npad)
        own[: r1 - r0] = v[r0 + perm]
        sends = {qq: own[np.asarray(reqs[qq][rank], dtype=np.int64)] for qq in range(G) if qq != rank}
        box = [None] * G
        dist.all_gather_object(box, sends)
        recv = np.zeros(H["n_halo"])
        for qq in range(G):
            if qq != rank:
                recv[off[qq]:off[qq + 1]] = box[qq][rank]
        xg = np.concatenate([own, recv])
        # logical column q * n_pad + p -> compact index (own: p; remote: n_pad + halo index)
        lookup = {}
        for qq in range(G):
            for t in range(off[qq], off[qq + 1]):
                lookup[qq * npad + int(hpos[t])] = npad + t
        ccol = np.array([c - rank * npad if c // npad == rank else lookup[int(c)] for c in col], dtype=np.int64)
        y = np.array([np.dot(val[rp[r]:rp[r + 1]], xg[ccol[rp[r]:rp[r + 1]]]) for r in range(r1 - r0)])
        yg = O.spmv(A.rowptr, A.col, A.val, v)[r0 + perm]
        # every remote column the rows touch is in the halo, nothing else is
        touched = {int(c) for c in col if c // npad != rank}
        q.put((rank, np.abs(y - yg).max() / max(1.0, np.abs(yg).max()), touched == set(lookup), int(H["n_halo"]),
               int(A.n - (r1 - r0))))
    finally:
        dist.destroy_process_group()


def test_two_rank_halo_exchange_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, exact_set, nhalo, nremote in out:
        assert err <= 1e-13, (rank, err)
        assert exact_set, f"rank {rank}: halo is not exactly the touched remote columns"
        assert 0 < nhalo < nremote  # the halo is smaller than the peer's whole slot


def _ingest_worker(rank, port, path, q):
    """Rank-local ingest (one process per GPU at C4 scale): rank 0 writes the matrix
    once (synthgen.save_csr), every rank maps it read-only, plans its own part from
    the mapped arrays, and the distributed symmetry check adds the ranks' hash sums
    over their own rows (topk_eig_plan_symmetry; create does this with NCCL)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import paper_2201_07498_b200 as T
        if rank == 0:
            S.save_csr(path, S.rmat(12, 40_000, 14))
        dist.barrier()
        A = S.load_csr_mmap(path)
        ref = S.rmat(12, 40_000, 14)
        same = (A.n == ref.n and np.array_equal(A.rowptr, ref.rowptr) and np.array_equal(A.col, ref.col)
                and np.array_equal(A.val, ref.val))
        G = WORLD
        b = T.plan_partition(np.asarray(A.rowptr), G)
        L = T.plan_layout(A, G, rank, "f64")
        Lr = T.plan_layout(ref, G, rank, "f64")
        layout_same = all(np.array_equal(L[k], Lr[k]) for k in ("rowptr", "col", "val", "perm"))

        def global_ok(M):
            mine = T.plan_symmetry(M, int(b[rank]), int(b[rank + 1]))
            allh = [torch.zeros(4, dtype=torch.int64) for _ in range(G)]
            dist.all_gather(allh, torch.from_numpy(mine.view(np.int64).copy()))
            tot = np.zeros(4, np.uint64)
            for t in allh:  # wrapping uint64 sums, rank order
                tot = tot + t.numpy().view(np.uint64)
            return bool(tot[0] == tot[2] and tot[1] == tot[3]), tot

        sym, tot = global_ok(A)
        whole = T.plan_symmetry(ref, 0, ref.n)
        # one asymmetric value (an entry in rank 1's rows): the summed check must fail
        bad = S.CSR(ref.n, ref.rowptr.copy(), ref.col.copy(), ref.val.copy())
        k = int(ref.rowptr[int(b[1])])
        bad.val[k] += 1.0 / 128
        asym, _ = global_ok(bad)
        q.put((rank, same, layout_same, sym, np.array_equal(tot, whole), asym))
    finally:
        dist.destroy_process_group()


def test_two_rank_shared_ingest_and_distributed_symmetry(tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "m.csr")
    procs = [ctx.Process(target=_ingest_worker, args=(r, port, path, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, layout_same, sym, whole_eq, asym in out:
        assert same, f"rank {rank}: mapped matrix differs"
        assert layout_same, f"rank {rank}: layout from the mapped arrays differs"
        assert sym and whole_eq, f"rank {rank}: distributed symmetry sums"
        assert not asym, f"rank {rank}: asymmetric value not detected"
