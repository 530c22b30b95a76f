// solver.cu — orchestrator and C ABI (include/topk_eig.h).
//
// One handle = one process's view: either a single process driving G row
// partitions on one device ("loopback": the G parts share the exchange buffers,
// so every exchange is a no-op ordered on one stream), or one rank of a
// multi-process NCCL job (one part per process, exchanges are in-place
// ncclAllGather over NVLink). Both run the same kernels in the same order, so a
// loopback-G solve and an NCCL-G solve are bitwise identical by construction.
//
// Per solve (DESIGN.md 8(a) a5-a15), all device-side, captured as ONE CUDA graph:
//   k_v1 -> [exchange] -> for i in 1..m: k_spmv, [x], k_step, [x], k_correct, [x]
//   -> k_jacobi -> k_ritz(pass 0: norms) -> [x] -> k_ritz(pass 1: output)
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <thread>

#include <omp.h>
#include <type_traits>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "host_prep.h"
#include "mem_pool.h"
#include "kernels.cuh"
#include "topk_eig.h"

using namespace topk;

static thread_local std::string g_last_error;

// TOPK_TRACE=1: stage timings of topk_eig_create on stderr (host-side profiling)
struct StageClock {
    bool on = false;
    std::chrono::steady_clock::time_point t0;
    StageClock() {
        const char *e = std::getenv("TOPK_TRACE");
        on = e && e[0] == '1';
        t0 = std::chrono::steady_clock::now();
    }
    void mark(const char *what) {
        if (!on) return;
        auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[topk create] %-28s %8.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

static topk_status_t fail(topk_status_t s, const std::string &msg) {
    g_last_error = msg;
    return s;
}

#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            throw CudaFail(std::string(#expr) + ": " + cudaGetErrorString(_e));              \
        }                                                                                    \
    } while (0)
#define NCCL_TRY(expr)                                                                       \
    do {                                                                                     \
        ncclResult_t _r = (expr);                                                            \
        if (_r != ncclSuccess) throw NcclFail(std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)

struct CudaFail { std::string msg; explicit CudaFail(std::string m) : msg(std::move(m)) {} };
struct NcclFail { std::string msg; explicit NcclFail(std::string m) : msg(std::move(m)) {} };

static size_t dsize(topk_dtype_t t) { return t == TOPK_F64 ? 8 : t == TOPK_F32 ? 4 : 2; }

// Host <-> device copy ordered on the handle's (non-blocking) stream and waited for:
// a plain cudaMemcpy runs on the legacy stream and would not wait for the stream's
// pending work (e.g. the zero fill of a freshly allocated block).
static cudaError_t scopy(cudaStream_t st, void *dst, const void *src, size_t n, cudaMemcpyKind k) {
    cudaError_t e = cudaMemcpyAsync(dst, src, n, k, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e;
}

struct SolveParams {
    uint64_t seed;
    int use_v1;
    int out_dtype;
    void *out_ptr;
};

// One SpMV pass on the device: physical arrays + work tables (host_prep.h).
struct SpmvDev {
    int nchunks = 0, nlong = 0, nitems = 0;
    int64_t nphys = 0;
    int32_t *col = nullptr;
    void *val = nullptr;
    Chunk *chunks = nullptr;
    LongRow *longrows = nullptr;
    int64_t *sell = nullptr;
    int32_t *items = nullptr;
    double *long_parts = nullptr, *alpha_long = nullptr;
    unsigned *long_cnt = nullptr;
    std::vector<int64_t> h_sell, h_bigptr;  // host copies (export_layout)
};

struct Part {
    int g = 0;
    int64_t row0 = 0, nrows = 0, npad = 0, nnz = 0;
    int nbig = 0;
    int64_t nnonempty = 0;
    int32_t *perm = nullptr;
    hvec<int32_t> h_perm;           // host copy: position -> part-local original row
    int32_t *inv = nullptr;         // original part-local row -> position
    hvec<int64_t> h_rowptr;         // host copy (export_layout)
    SpmvDev sp;                     // the SpMV (final pass when split)
    SpmvDev own;                    // two-pass SpMV: own-slot columns first
    double *ypart = nullptr;        // own-slot row sums of the first pass (nullptr: one pass)
    int32_t *owndeg = nullptr;      // own-slot entries per position (device; export_layout)
    void *yt = nullptr;            // Ritz output in position order, K values per row
    void *Vs = nullptr;            // thick restart scratch: keep columns (reading Q26)
    int *pro_gate = nullptr, *pro_force = nullptr, *pro_count = nullptr;  // reading Q29 (state ints)
    double *pro_w = nullptr;       // [3][m + 2] orthogonality estimates
    // halo exchange (reading Q27): compact SpMV input x_g = [own slot | remote entries]
    void *xg = nullptr;
    int64_t nhalo = 0;
    std::vector<int64_t> halo_off;     // G+1 (host)
    std::vector<int32_t> halo_pos_h;   // remote entry -> owner position (host, exports)
    int32_t *halo_q = nullptr, *halo_pos = nullptr;  // device (pull)
    std::vector<int64_t> send_off;     // G+1 (multi-process)
    int32_t *send_pos = nullptr;       // device: own positions requested by each peer
    void *sendbuf = nullptr;
    void *V = nullptr, *y = nullptr, *w = nullptr;
    void *out = nullptr;       // internal eigenvector output (K * nrows f64)
    double *v1buf = nullptr;
    double *y_dbg = nullptr;
    double *slots = nullptr;
    unsigned *counters = nullptr;  // [8]
    char *state = nullptr;         // device state block
    size_t state_bytes = 0;
    LzState st{};
    std::vector<char> hstate;      // host mirror
};

struct topk_eig_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int64_t n = 0;
    int K = 0, m = 0, G = 1, world = 1, rank = 0;
    topk_dtype_t vs = TOPK_F64, ms = TOPK_F64, cs = TOPK_F64;
    int reorth = 1;
    double tau = 1e-12;
    double conv_tol = 0.0;   // reading Q25 (0: fixed m)
    int keep = 0;            // reading Q26: Ritz pairs kept per thick restart (0: off)
    int period = 1;          // reading Q28: reorthogonalise every period-th iteration
    int max_restarts = 0;
    int conv_check = 0;      // check period c
    int conv_checks = 0;     // checks enqueued per solve
    int use_graph = 1;
    int nsm = 148;
    int grid_spmv_v[2] = {0, 0};  // k_spmv without / with the big-row chunk path
    int grid_spmv = 0, grid_stream = 0, grid_step = 0, grid_corr = 0, grid_ritz = 0;
    int ritz_tn = 0;           // > 0: Ritz output pass on the fp64 tensor cores, 8 * ritz_tn outputs per warp
    bool use_gram = false;  // Ritz norms from the Gram matrix (reading Q24; no Ritz pass 0)
    int grid_stepw[kStepMaxNC + 1] = {0};
    int grid_corrw[kCorrMaxNC + 1] = {0};
#ifdef TOPK_NO_CORRW
    bool corrw = false;                // dev build variant: k_correct at every width
#else
    bool corrw = true;                 // exact-width correction for it <= kCorrMaxNC
#endif
    bool restart_unrolled = false;     // opts.restart_loop = 1: unrolled restart cycles, no WHILE node
    int ritz_mode = 0;                 // opts.ritz_path: 0 auto, 1 fp64 CUDA cores only
    std::vector<int64_t> bounds;
    std::vector<Part> parts;
    Exch ex{};
    char *exch_block = nullptr;
    void *replica = nullptr;
    bool halo = false;                 // opts.exchange == 1 (reading Q27)
    cudaStream_t body_stream = nullptr; // captures the thick-restart WHILE body (reading Q26)
    bool split = false;                // two-pass SpMV: own-slot columns first
    cudaStream_t comm_stream = nullptr; // one process per GPU + split: the vector exchange overlaps
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool join_pending = false;
    const void **d_xsrc = nullptr;     // device: every local part's x_g (halo pull)
    SolveParams *dparams = nullptr, *hparams = nullptr;  // hparams: pageable (a pinned block's free
                                                          // measured up to 380 ms on destroy)
    std::vector<SolveParams> hparams_own;
    double *jac_work = nullptr;
    size_t jac_smem = 0, jac_bytes = 0;
    int jac_ld_log2 = 0, jac_hl_log2 = 0;

    int jac_threads = 32;
    int jac_cl = 0;            // cluster size of k_jacobi_cl (0: single-CTA k_jacobi)
    size_t jac_cl_smem = 0;
    cudaGraphExec_t gexec = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t evL = nullptr, evJ = nullptr;  // end of the Lanczos phase / of the final Jacobi (info ms_*)
    int64_t bytes_nvlink = 0;                  // modelled bytes received over the interconnect per solve
    ncclComm_t comm = nullptr;
    bool sticky = false;
    int64_t bytes_model = 0;
    int64_t launches = 0;
    int profile = 0;
    bool capturing = false;
    struct Prof { int cls; cudaEvent_t a, b; };
    std::vector<Prof> prof;
    size_t prof_next = 0;
    void (*enqueue)(topk_eig_s *, bool) = nullptr;
    void (*spmv_only)(topk_eig_s *, Part &) = nullptr;
    std::vector<void *> allocs;

    topk_eig_s() = default;
    topk_eig_s(const topk_eig_s &) = delete;
    topk_eig_s &operator=(const topk_eig_s &) = delete;
    // Releases everything the handle owns, also after a failed create (any prefix of
    // the set-up): graph, NCCL comm, pool blocks, events, streams.
    ~topk_eig_s();

    template <typename T> T *alloc(size_t count) {
        size_t bytes = std::max<size_t>(count * sizeof(T), 256);
        void *p = pool_dev_alloc(bytes);  // caching allocator (mem_pool.h)
        if (!p) CUDA_TRY(cudaErrorMemoryAllocation);
        allocs.push_back(p);
        CUDA_TRY(cudaMemsetAsync(p, 0, bytes, stream));
        return reinterpret_cast<T *>(p);
    }
};

// ---------------------------------------------------------------------------
// per-kernel-class event brackets (part 0 only); inside a capture they become
// external event-record nodes of the graph
static void prof_begin(topk_eig_s *h, const Part &p, int cls) {
    if (!h->profile || &p != &h->parts[0]) return;
    if (h->prof_next == h->prof.size()) {
        topk_eig_s::Prof q{cls, nullptr, nullptr};
        CUDA_TRY(cudaEventCreate(&q.a));
        CUDA_TRY(cudaEventCreate(&q.b));
        h->prof.push_back(q);
    }
    topk_eig_s::Prof &q = h->prof[h->prof_next];
    q.cls = cls;
    if (h->capturing) CUDA_TRY(cudaEventRecordWithFlags(q.a, h->stream, cudaEventRecordExternal));
    else CUDA_TRY(cudaEventRecord(q.a, h->stream));
}
static void prof_end(topk_eig_s *h, const Part &p) {
    if (!h->profile || &p != &h->parts[0]) return;
    topk_eig_s::Prof &q = h->prof[h->prof_next++];
    if (h->capturing) CUDA_TRY(cudaEventRecordWithFlags(q.b, h->stream, cudaEventRecordExternal));
    else CUDA_TRY(cudaEventRecord(q.b, h->stream));
}

// ---------------------------------------------------------------------------
// exchanges (no-ops in loopback: shared buffers on one stream)
static void exch_join(topk_eig_s *h);
static void launch_jacobi(topk_eig_s *h, int check) {
    exch_join(h);  // beta_{i+1} comes from the exchanged norm partials
    for (Part &p : h->parts) {
        JacArgs a;
        a.st = p.st; a.ex = h->ex; a.G = h->G; a.m = h->m; a.K = h->K; a.max_sweeps = 50;
        a.work = h->jac_work ? h->jac_work + (size_t)(&p - &h->parts[0]) * (h->jac_bytes / 8) : nullptr;
        a.ld_log2 = h->jac_ld_log2;
        a.hl_log2 = h->jac_hl_log2;
        a.check = check;
        a.conv_tol = h->conv_tol;
        a.max_restarts = h->max_restarts;
        prof_begin(h, p, 4);
        if (h->jac_cl > 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)h->jac_cl);
            cfg.blockDim = dim3(kJacClNT);
            cfg.dynamicSmemBytes = h->jac_cl_smem;
            cfg.stream = h->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)h->jac_cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CUDA_TRY(cudaLaunchKernelEx(&cfg, k_jacobi_cl, a));
        } else if (h->jac_work) {
            k_jacobi<false><<<1, h->jac_threads, 0, h->stream>>>(a);
        } else {
            k_jacobi<true><<<1, h->jac_threads, h->jac_smem, h->stream>>>(a);
        }
        CUDA_TRY(cudaGetLastError());
        prof_end(h, p);
        h->launches++;
    }
}

// halo exchange of the current vector (reading Q27): parts on one device pull their
// remote entries; one process per GPU packs what each peer asked for and exchanges it
// with grouped NCCL send/recv straight into the peers' compact vectors
static void exch_halo(topk_eig_s *h) {
    const size_t es = dsize(h->vs);
    auto launch_pull = [&](Part &p) {
        if (p.nhalo == 0) return;
        const unsigned grid = (unsigned)std::min<int64_t>((p.nhalo + 255) / 256, (int64_t)h->nsm * 8);
        if (es == 8) k_halo_pull<uint64_t><<<grid, 256, 0, h->stream>>>((uint64_t *)p.xg, p.npad, p.nhalo, p.halo_q, p.halo_pos, (const uint64_t *const *)h->d_xsrc);
        else if (es == 4) k_halo_pull<uint32_t><<<grid, 256, 0, h->stream>>>((uint32_t *)p.xg, p.npad, p.nhalo, p.halo_q, p.halo_pos, (const uint32_t *const *)h->d_xsrc);
        else k_halo_pull<uint16_t><<<grid, 256, 0, h->stream>>>((uint16_t *)p.xg, p.npad, p.nhalo, p.halo_q, p.halo_pos, (const uint16_t *const *)h->d_xsrc);
        CUDA_TRY(cudaGetLastError());
        h->launches++;
    };
    if (!h->comm) {
        for (Part &p : h->parts) launch_pull(p);
        return;
    }
    Part &p = h->parts[0];
    const int64_t nsend = p.send_off.back();
    if (nsend > 0) {
        const unsigned grid = (unsigned)std::min<int64_t>((nsend + 255) / 256, (int64_t)h->nsm * 8);
        if (es == 8) k_halo_pack<uint64_t><<<grid, 256, 0, h->stream>>>((const uint64_t *)p.xg, nsend, p.send_pos, (uint64_t *)p.sendbuf);
        else if (es == 4) k_halo_pack<uint32_t><<<grid, 256, 0, h->stream>>>((const uint32_t *)p.xg, nsend, p.send_pos, (uint32_t *)p.sendbuf);
        else k_halo_pack<uint16_t><<<grid, 256, 0, h->stream>>>((const uint16_t *)p.xg, nsend, p.send_pos, (uint16_t *)p.sendbuf);
        CUDA_TRY(cudaGetLastError());
        h->launches++;
    }
    NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < h->G; ++q) {
        if (q == h->rank) continue;
        const size_t ns = (size_t)(p.send_off[(size_t)q + 1] - p.send_off[(size_t)q]);
        const size_t nr = (size_t)(p.halo_off[(size_t)q + 1] - p.halo_off[(size_t)q]);
        if (ns) NCCL_TRY(ncclSend((char *)p.sendbuf + (size_t)p.send_off[(size_t)q] * es, ns * es, ncclUint8, q, h->comm, h->stream));
        if (nr) NCCL_TRY(ncclRecv((char *)p.xg + (size_t)(p.npad + p.halo_off[(size_t)q]) * es, nr * es, ncclUint8, q, h->comm, h->stream));
    }
    NCCL_TRY(ncclGroupEnd());
}

static void exch_vec_norm(topk_eig_s *h) {
    exch_join(h);
    if (h->halo) {
        exch_halo(h);
        if (h->comm) NCCL_TRY(ncclAllGather(h->ex.norm_part + h->rank, h->ex.norm_part, 1, ncclFloat64, h->comm, h->stream));
        return;
    }
    if (!h->comm) return;
    Part &p = h->parts[0];
    size_t vb = (size_t)p.npad * dsize(h->vs);
    // two-pass SpMV: the vector (and the norm partials) move on the comm stream while the
    // next SpMV's own-slot pass runs; launch_spmv joins before its final pass
    cudaStream_t cs = h->stream;
    if (h->split && h->comm_stream) {
        CUDA_TRY(cudaEventRecord(h->ev_fork, h->stream));
        CUDA_TRY(cudaStreamWaitEvent(h->comm_stream, h->ev_fork, 0));
        cs = h->comm_stream;
    }
    NCCL_TRY(ncclGroupStart());
    NCCL_TRY(ncclAllGather((char *)h->replica + (size_t)h->rank * vb, h->replica, vb, ncclUint8, h->comm, cs));
    NCCL_TRY(ncclAllGather(h->ex.norm_part + h->rank, h->ex.norm_part, 1, ncclFloat64, h->comm, cs));
    NCCL_TRY(ncclGroupEnd());
    if (cs != h->stream) {
        CUDA_TRY(cudaEventRecord(h->ev_join, cs));
        h->join_pending = true;
    }
}
// the main stream waits for an exchange still running on the comm stream
static void exch_join(topk_eig_s *h) {
    if (!h->join_pending) return;
    CUDA_TRY(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
    h->join_pending = false;
}
static void exch_norm(topk_eig_s *h) {
    exch_join(h);  // one NCCL operation of the communicator at a time
    if (!h->comm) return;
    NCCL_TRY(ncclAllGather(h->ex.norm_part + h->rank, h->ex.norm_part, 1, ncclFloat64, h->comm, h->stream));
}
static void exch_alpha(topk_eig_s *h) {
    exch_join(h);  // one NCCL operation of the communicator at a time
    if (!h->comm) return;
    NCCL_TRY(ncclAllGather(h->ex.alpha_part + h->rank, h->ex.alpha_part, 1, ncclFloat64, h->comm, h->stream));
}
static void exch_h(topk_eig_s *h) {
    exch_join(h);  // one NCCL operation of the communicator at a time
    if (!h->comm) return;
    size_t ld = (size_t)h->m + 1;
    NCCL_TRY(ncclAllGather(h->ex.hpart + h->rank * 2 * ld, h->ex.hpart, 2 * ld, ncclFloat64, h->comm, h->stream));
}
static void exch_ritz(topk_eig_s *h) {
    exch_join(h);  // one NCCL operation of the communicator at a time
    if (!h->comm) return;
    NCCL_TRY(ncclAllGather(h->ex.ritz_part + (size_t)h->rank * h->K, h->ex.ritz_part, h->K, ncclFloat64, h->comm, h->stream));
}

static void *rep_slot(topk_eig_s *h, Part &p) {
    if (h->G == 1) return nullptr;
    if (h->halo) return p.xg;  // own slot of the compact vector
    return (char *)h->replica + (size_t)p.g * p.npad * dsize(h->vs);
}

// ---------------------------------------------------------------------------
static void pass_args(SpmvArgs &a, const SpmvDev &d) {
    a.col = d.col; a.val = d.val;
    a.chunks = d.chunks; a.longrows = reinterpret_cast<const int4 *>(d.longrows);
    a.sell = reinterpret_cast<const longlong2 *>(d.sell); a.items = reinterpret_cast<const int2 *>(d.items);
    a.nchunks = d.nchunks; a.nitems = d.nitems;
    a.long_parts = d.long_parts; a.long_cnt = d.long_cnt;
    a.alpha_long = d.alpha_long; a.nlong = d.nlong;
}

template <typename VT, typename ST, typename CT, bool LOCAL>
static void spmv_pass(topk_eig_s *h, const SpmvArgs &a, int it) {
    if (a.nchunks > 0)
        k_spmv<VT, ST, CT, LOCAL><<<h->grid_spmv_v[1], kSpmvNT, 0, h->stream>>>(a, it);
    else
        k_spmv_sell<VT, ST, CT, LOCAL><<<h->grid_spmv_v[0], kSpmvNT, 0, h->stream>>>(a, it);
    CUDA_TRY(cudaGetLastError());
}

// a7. Two-pass SpMV (h->split): the own-slot columns first (they do
// not need the vector exchange), then -- after the exchange, which one process per GPU
// runs on the comm stream meanwhile -- the other columns plus the epilogue.
template <typename VT, typename ST, typename CT>
static void launch_spmv(topk_eig_s *h, Part &p, int it, double *y_dbg) {
    SpmvArgs a;
    a.nbig = p.nbig; a.nnonempty = (int)p.nnonempty;
    const void *ucol = (const char *)p.V + (size_t)(it - 1) * p.npad * sizeof(ST);
    a.x = (h->G == 1) ? ucol : (h->halo ? p.xg : h->replica);
    a.xlen = (h->G == 1) ? p.npad : (h->halo ? p.npad + p.nhalo : (int64_t)h->G * p.npad);
    a.ui = ucol;
    a.y = p.y; a.y_dbg = y_dbg;
    a.ypart = p.ypart;
    a.slots = p.slots; a.counter = p.counters + 1;
    a.st = p.st; a.ex = h->ex; a.G = h->G; a.g = p.g;
    prof_begin(h, p, 1);
    if (p.ypart) {
        pass_args(a, p.own);
        spmv_pass<VT, ST, CT, true>(h, a, it);
        h->launches++;
        exch_join(h);  // the remote columns need the exchanged vector
    }
    pass_args(a, p.sp);
    spmv_pass<VT, ST, CT, false>(h, a, it);
    prof_end(h, p);
    h->launches++;
}

template <typename ST, typename CT, int NC>
static void stepw_one(topk_eig_s *h, const StepArgs &a, int it, int j0) {
    k_stepw<ST, CT, NC><<<h->grid_stepw[NC], kNT, 0, h->stream>>>(a, it, j0);
    CUDA_TRY(cudaGetLastError());
}
template <typename ST, typename CT, int NC>
static void stepw_dispatch(topk_eig_s *h, const StepArgs &a, int it, int j0, int width) {
    if constexpr (NC > kStepMaxNC) {
        throw CudaFail("multi-dot pass wider than kStepMaxNC");
    } else {
        if (width == NC) stepw_one<ST, CT, NC>(h, a, it, j0);
        else stepw_dispatch<ST, CT, NC + 1>(h, a, it, j0, width);
    }
}
template <typename ST, typename CT>
static void launch_stepw(topk_eig_s *h, const StepArgs &a, int it, int j0, int width) {
    stepw_dispatch<ST, CT, 1>(h, a, it, j0, width);
}
template <typename ST, typename CT, int NC>
static void stepw_grids(topk_eig_s *h) {
    if constexpr (NC <= kStepMaxNC) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_stepw<ST, CT, NC>, kNT, 0);
        h->grid_stepw[NC] = h->nsm * std::max(1, std::min(occ, 8));
        stepw_grids<ST, CT, NC + 1>(h);
    }
}

template <typename ST, typename CT>
static void launch_step(topk_eig_s *h, Part &p, int it, int mode, int no_prev = 0, const int *gate = nullptr) {
    StepArgs a;
    a.no_prev = no_prev;
    a.gate = gate;
    a.y = p.y; a.w = p.w; a.V = p.V;
    a.vout = (char *)p.V + (size_t)it * p.npad * sizeof(ST);
    a.rep_slot = (mode == 1) ? rep_slot(h, p) : nullptr;
    a.npad = p.npad; a.ld = h->m + 1;
    a.slots = p.slots; a.counter = p.counters + 2;
    a.st = p.st; a.ex = h->ex; a.G = h->G; a.g = p.g; a.mode = mode;
    prof_begin(h, p, 2);
    if (mode == 1) {  // reorth off: recurrence + publish only
        k_step<ST, CT, kStepJB><<<h->grid_step, kNT, 0, h->stream>>>(a, it);
        CUDA_TRY(cudaGetLastError());
        h->launches++;
    } else {
        // exact-width passes: one pass up to 17 columns, else balanced passes of <= 16
        const int npass = (it <= kStepMaxNC) ? 1 : (it + 15) / 16;
        int j0 = 0;
        for (int ps = 0; ps < npass; ++ps) {
            const int width = (it - j0 + (npass - ps) - 1) / (npass - ps);
            launch_stepw<ST, CT>(h, a, it, j0, width);
            j0 += width;
            h->launches++;
        }
    }
    prof_end(h, p);
}

template <typename ST, typename CT, int NC>
static void correctw_dispatch(topk_eig_s *h, const CorrArgs &a, int it, size_t smem) {
    if constexpr (NC > kCorrMaxNC) {
        throw CudaFail("exact-width correction wider than kCorrMaxNC");
    } else {
        if (it == NC) {
            k_correctw<ST, CT, NC><<<h->grid_corrw[NC], kNT, smem, h->stream>>>(a, it);
            CUDA_TRY(cudaGetLastError());
        } else {
            correctw_dispatch<ST, CT, NC + 1>(h, a, it, smem);
        }
    }
}
template <typename ST, typename CT, int NC>
static void correctw_grids(topk_eig_s *h) {
    if constexpr (NC <= kCorrMaxNC) {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_correctw<ST, CT, NC>, kNT, (size_t)3 * (h->m + 1) * 8);
        h->grid_corrw[NC] = h->nsm * std::max(1, std::min(occ, 8));
        correctw_grids<ST, CT, NC + 1>(h);
    }
}

template <typename ST, typename CT>
static void launch_correct(topk_eig_s *h, Part &p, int it, int in_col, const int *gate = nullptr) {
    CorrArgs a;
    a.gate = gate;
    a.w = p.w; a.V = p.V; a.rep_slot = rep_slot(h, p);
    a.npad = p.npad; a.ld = h->m + 1;
    a.slots = p.slots; a.counter = p.counters + 3;
    a.st = p.st; a.ex = h->ex; a.G = h->G; a.g = p.g; a.in_col = in_col;
    size_t smem = (size_t)3 * (h->m + 1) * sizeof(double);
    prof_begin(h, p, 3);
    // the register-pipelined correction measured faster than a TMA (cp.async.bulk +
    // mbarrier) ring (57 vs 75 us at it = 17, gpurun_out/r01n; that variant was removed)
    if (it <= kCorrMaxNC && h->corrw)
        correctw_dispatch<ST, CT, 1>(h, a, it, smem);  // exact-width: all it basis loads in flight
    else
        k_correct<ST, CT><<<h->grid_corr, kNT, smem, h->stream>>>(a, it);
    CUDA_TRY(cudaGetLastError());
    prof_end(h, p);
    h->launches++;
}

// thick restart (reading Q26): Jacobi on the cycle's T (convergence test + the
// kept pairs), projection of the kept Ritz vectors, norm exchange, basis rewrite
static void exch_rst(topk_eig_s *h) {
    exch_join(h);  // one NCCL operation of the communicator at a time
    if (!h->comm) return;
    NCCL_TRY(ncclAllGather(h->ex.rst_part + (size_t)h->rank * h->keep, h->ex.rst_part, h->keep, ncclFloat64,
                           h->comm, h->stream));
}
template <typename ST, typename CT>
static void launch_restart(topk_eig_s *h, bool decide = true) {
    if (decide) launch_jacobi(h, 2);  // the restart data (or the converged stop)
    const int ng = (h->keep + kRitzKB - 1) / kRitzKB;
    for (Part &p : h->parts) {
        RestartArgs a;
        a.V = p.V; a.Vs = p.Vs; a.npad = p.npad; a.keep = h->keep; a.G = h->G; a.g = p.g; a.mm = h->m;
        a.slots = p.slots; a.counter = p.counters + 8;
        a.st = p.st; a.ex = h->ex;
        const int nrb = std::max(1, h->grid_ritz / ng);
        const size_t smem = (size_t)h->m * kRitzKB * sizeof(CT);
        prof_begin(h, p, 5);
        k_restart_proj<ST, CT, kRitzKB><<<nrb * ng, kNT, smem, h->stream>>>(a);
        CUDA_TRY(cudaGetLastError());
        prof_end(h, p);
        h->launches++;
    }
    exch_rst(h);
    for (Part &p : h->parts) {
        RestartArgs a;
        a.V = p.V; a.Vs = p.Vs; a.npad = p.npad; a.keep = h->keep; a.G = h->G; a.g = p.g; a.mm = h->m;
        a.slots = p.slots; a.counter = p.counters + 8;
        a.st = p.st; a.ex = h->ex;
        prof_begin(h, p, 5);
        k_restart_copy<ST><<<h->grid_stream, kNT, 0, h->stream>>>(a);
        CUDA_TRY(cudaGetLastError());
        prof_end(h, p);
        h->launches++;
    }
}

static void launch_pro(topk_eig_s *h, Part &p, int it) {
    ProArgs a;
    a.st = p.st; a.ex = h->ex; a.G = h->G;
    a.eps = h->vs == TOPK_F64 ? std::ldexp(1.0, -53) : h->vs == TOPK_F32 ? std::ldexp(1.0, -24) : std::ldexp(1.0, -8);
    a.psi = a.eps * std::sqrt((double)h->n);
    a.W = p.pro_w; a.gate = p.pro_gate; a.force = p.pro_force; a.count = p.pro_count;
    k_pro<<<1, 256, 0, h->stream>>>(a, it);
    CUDA_TRY(cudaGetLastError());
    h->launches++;
}

// phase boundary events (topk_eig_info_t ms_lanczos / ms_jacobi / ms_ritz): event-record
// nodes when the solve is being captured
static void record_event(topk_eig_s *h, cudaEvent_t e) {
    if (h->capturing) CUDA_TRY(cudaEventRecordWithFlags(e, h->stream, cudaEventRecordExternal));
    else CUDA_TRY(cudaEventRecord(e, h->stream));
}

// a14 output pass on the fp64 tensor cores (k_ritz_mma; compute dtype f64 only)
template <typename ST, int TN>
static void ritz_mma_tn(topk_eig_s *h, const RitzArgs &a) {
    const int nog = (h->K + 8 * TN - 1) / (8 * TN);
    const size_t smem = ((size_t)((h->m + 3) & ~3) * 8 * TN + 8 * TN) * sizeof(double);
    k_ritz_mma<ST, TN><<<(unsigned)(h->nsm * 2 * nog), kNT, smem, h->stream>>>(a);
}
template <typename ST, typename CT>
static void launch_ritz_mma(topk_eig_s *h, const RitzArgs &a) {
    if constexpr (std::is_same<CT, double>::value) {
        switch (h->ritz_tn) {
            case 1: ritz_mma_tn<ST, 1>(h, a); break;
            case 2: ritz_mma_tn<ST, 2>(h, a); break;
            case 3: ritz_mma_tn<ST, 3>(h, a); break;
            default: ritz_mma_tn<ST, 4>(h, a); break;
        }
    } else {
        throw CudaFail("k_ritz_mma needs compute dtype f64");
    }
}

template <typename VT, typename ST, typename CT>
static void enqueue_solve(topk_eig_s *h, bool want_vectors) {
    // a5: v1
    for (Part &p : h->parts) {
        V1Args a;
        a.u0 = p.V; a.rep_slot = rep_slot(h, p);
        a.seed = &h->dparams->seed; a.use_v1 = &h->dparams->use_v1; a.v1 = p.v1buf; a.perm = p.perm;
        a.row0 = p.row0; a.nrows = p.nrows; a.npad = p.npad;
        a.slots = p.slots; a.counter = p.counters + 0;
        a.st = p.st; a.ex = h->ex; a.g = p.g;
        prof_begin(h, p, 0);
        k_v1<ST, CT><<<h->grid_stream, kNT, 0, h->stream>>>(a);
        CUDA_TRY(cudaGetLastError());
        prof_end(h, p);
        h->launches++;
    }
    exch_vec_norm(h);
    // cycles: the paper's fixed m iterations (cycle 0 only), or thick-restart cycles
    // (reading Q26): restart after cycles 0 .. R-1, then steps keep+1 .. m again
    const int R = h->keep > 0 ? h->max_restarts : 0;
    // reading Q25: the convergence check follows iteration it whatever kind of step it was
    auto maybe_check = [&](int it) {
        if (h->keep == 0 && h->conv_tol > 0.0 && it >= h->K && it < h->m && it % h->conv_check == 0)
            launch_jacobi(h, 1);  // may set done = 2 (later launches return at once)
    };
    auto run_cycle = [&](int cyc) {
    const int it0 = (cyc == 0) ? 1 : h->keep + 1;
    for (int it = it0; it <= h->m; ++it) {
        for (Part &p : h->parts) launch_spmv<VT, ST, CT>(h, p, it, nullptr);
        exch_alpha(h);
        if (h->reorth == 3) {
            // partial reorthogonalisation (reading Q29): three-term step, Simon's estimate,
            // then the gated second pass (dots of u_{i+1} against V, correction in place)
            for (Part &p : h->parts) launch_step<ST, CT>(h, p, it, 1);
            exch_norm(h);
            for (Part &p : h->parts) launch_pro(h, p, it);
            for (Part &p : h->parts) launch_step<ST, CT>(h, p, it, 2, 0, p.pro_gate);
            exch_h(h);
            for (Part &p : h->parts) launch_correct<ST, CT>(h, p, it, it, p.pro_gate);
            exch_vec_norm(h);
            maybe_check(it);
            continue;
        }
        // reorth off (the paper's optional mode), or an iteration between two periodic
        // reorthogonalisations (reading Q28): the three-term step publishes u_{i+1}
        if (h->reorth < 0 || (h->period > 1 && it % h->period != 0 && (it == 1 || (it - 1) % h->period != 0))) {
            for (Part &p : h->parts) launch_step<ST, CT>(h, p, it, 1);
            exch_vec_norm(h);
            maybe_check(it);
            continue;
        }
        for (Part &p : h->parts) launch_step<ST, CT>(h, p, it, 0, (cyc > 0 && it == it0) ? 1 : 0);
        exch_h(h);
        for (Part &p : h->parts) launch_correct<ST, CT>(h, p, it, -1);
        if (h->reorth == 2) {
            exch_norm(h);
            for (Part &p : h->parts) launch_step<ST, CT>(h, p, it, 2);
            exch_h(h);
            for (Part &p : h->parts) launch_correct<ST, CT>(h, p, it, it);
        }
        exch_vec_norm(h);
        maybe_check(it);
    }
    };
    // thick restart inside a captured graph: cycle 0, then a WHILE node whose body is one
    // restart + cycle, looping on the device (no unrolled cycles, no host round trip).
    // Unrolled cycles (finished ones return at once) when not capturing, when profiling
    // (event nodes are not allowed in conditional bodies), with several processes, or
    // with opts.restart_loop = 1.
    const bool use_while = R > 0 && h->capturing && !h->profile && h->world == 1 && !h->restart_unrolled;
    if (!use_while) {
        for (int cyc = 0; cyc <= R; ++cyc) {
            run_cycle(cyc);
            if (cyc < R) launch_restart<ST, CT>(h);
        }
    } else {
        run_cycle(0);
        launch_jacobi(h, 2);
        cudaStreamCaptureStatus cs;
        cudaGraph_t g = nullptr;
        const cudaGraphNode_t *deps = nullptr;
        size_t ndep = 0;
        CUDA_TRY(cudaStreamGetCaptureInfo(h->stream, &cs, nullptr, &g, &deps, &ndep));
        cudaGraphConditionalHandle ch;
        CUDA_TRY(cudaGraphConditionalHandleCreate(&ch, g, 0, 0));
        Part &p0 = h->parts[0];
        k_restart_cond<<<1, 32, 0, h->stream>>>(ch, p0.st.done, p0.st.restarts, R);
        CUDA_TRY(cudaGetLastError());
        h->launches++;
        CUDA_TRY(cudaStreamGetCaptureInfo(h->stream, &cs, nullptr, &g, &deps, &ndep));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = ch;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        CUDA_TRY(cudaGraphAddNode(&cn, g, deps, ndep, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CUDA_TRY(cudaStreamUpdateCaptureDependencies(h->stream, &cn, 1, cudaStreamSetCaptureDependencies));
        if (!h->body_stream) CUDA_TRY(cudaStreamCreateWithFlags(&h->body_stream, cudaStreamNonBlocking));
        cudaStream_t main_stream = h->stream;
        CUDA_TRY(cudaStreamBeginCaptureToGraph(h->body_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        h->stream = h->body_stream;
        try {
            launch_restart<ST, CT>(h, false);
            run_cycle(1);
            launch_jacobi(h, 2);
            k_restart_cond<<<1, 32, 0, h->stream>>>(ch, p0.st.done, p0.st.restarts, R);
            CUDA_TRY(cudaGetLastError());
            h->launches++;
        } catch (...) {
            h->stream = main_stream;
            cudaGraph_t dummy;
            cudaStreamEndCapture(h->body_stream, &dummy);
            throw;
        }
        h->stream = main_stream;
        cudaGraph_t body_out;
        CUDA_TRY(cudaStreamEndCapture(h->body_stream, &body_out));
    }
    // a12-a13: Jacobi (redundant on every part, identical inputs)
    exch_join(h);
    record_event(h, h->evL);
    launch_jacobi(h, 0);
    record_event(h, h->evJ);
    if (!want_vectors) return;
    // a14: Ritz projection + normalisation, two streaming passes (norms, output)
    for (int pass = h->use_gram ? 1 : 0; pass < 2; ++pass) {
        for (Part &p : h->parts) {
            RitzArgs a;
            a.V = p.V; a.npad = p.npad; a.nrows = p.nrows; a.K = h->K; a.G = h->G; a.g = p.g;
            a.slots = p.slots; a.counter = p.counters + 8;
            a.st = p.st; a.ex = h->ex;
            a.out_ptr = (void *const *)((char *)h->dparams + sizeof(SolveParams) * (1 + (&p - &h->parts[0])) +
                                        offsetof(SolveParams, out_ptr));
            a.out_dtype = &h->dparams->out_dtype;
            a.yt = p.yt;
            const size_t smem = (size_t)h->m * kRitzKB * sizeof(double);
            const unsigned ngroups = (unsigned)((h->K + kRitzKB - 1) / kRitzKB);
            const dim3 grid((unsigned)h->grid_ritz * ngroups);
            prof_begin(h, p, 5 + pass);
            if (pass == 1 && h->ritz_tn > 0) launch_ritz_mma<ST, CT>(h, a);
            else if (pass == 0) k_ritz<ST, CT, kRitzKB, 0><<<grid, kNT, smem, h->stream>>>(a);
            else k_ritz<ST, CT, kRitzKB, 1><<<grid, kNT, smem, h->stream>>>(a);
            CUDA_TRY(cudaGetLastError());
            prof_end(h, p);
            h->launches++;
        }
        if (pass == 0) exch_ritz(h);
    }
    // a15 prep: position order -> original row order into the caller's buffer
    for (Part &p : h->parts) {
        UnpermArgs a;
        a.yt = p.yt; a.inv = p.inv; a.nrows = p.nrows; a.npad = p.npad; a.K = h->K; a.k_found = p.st.k_found;
        a.out_ptr = (void *const *)((char *)h->dparams + sizeof(SolveParams) * (1 + (&p - &h->parts[0])) +
                                    offsetof(SolveParams, out_ptr));
        a.out_dtype = &h->dparams->out_dtype;
        prof_begin(h, p, 7);
        k_unperm<<<h->grid_stream, kNT, 0, h->stream>>>(a);
        CUDA_TRY(cudaGetLastError());
        prof_end(h, p);
        h->launches++;
    }
}

template <typename VT, typename ST, typename CT>
static void spmv_only(topk_eig_s *h, Part &p) {
    launch_spmv<VT, ST, CT>(h, p, 1, p.y_dbg);
}

template <typename VT, typename ST, typename CT>
static void set_kernels(topk_eig_s *h) {
    h->enqueue = &enqueue_solve<VT, ST, CT>;
    h->spmv_only = &spmv_only<VT, ST, CT>;
    int occ = 0;
    // the SpMV uses no dynamic shared memory: the whole unified L1 caches x
    CUDA_TRY(cudaFuncSetAttribute(k_spmv<VT, ST, CT, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CUDA_TRY(cudaFuncSetAttribute(k_spmv<VT, ST, CT, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CUDA_TRY(cudaFuncSetAttribute(k_spmv_sell<VT, ST, CT, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CUDA_TRY(cudaFuncSetAttribute(k_spmv_sell<VT, ST, CT, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv<VT, ST, CT, false>, kSpmvNT, 0);
    h->grid_spmv_v[1] = h->nsm * std::max(1, occ);
    occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_spmv_sell<VT, ST, CT, false>, kSpmvNT, 0);
    h->grid_spmv_v[0] = h->nsm * std::max(1, occ);
    h->grid_spmv = std::max(h->grid_spmv_v[0], h->grid_spmv_v[1]);  // slot allocation
    int occ2 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, k_step<ST, CT, kStepJB>, kNT, 0);
    h->grid_step = h->nsm * std::max(1, std::min(occ2, 8));
    int occ4 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ4, k_correct<ST, CT>, kNT, (size_t)3 * (h->m + 1) * sizeof(double));
    h->grid_corr = h->nsm * std::max(1, std::min(occ4, 8));
    h->grid_stream = h->nsm * 4;
    stepw_grids<ST, CT, 1>(h);
    correctw_grids<ST, CT, 1>(h);
    // Ritz norms from the Gram matrix (k_correct recursion) whenever dots are computed;
    // restarts replace basis columns and periodic reorth skips the dots: explicit norm pass
    h->use_gram = (h->reorth == 1 || h->reorth == 2) && h->keep == 0 && h->period == 1;
    int occ3 = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ3, k_ritz<ST, CT, kRitzKB, 1>, kNT, (size_t)h->m * kRitzKB * 8);
    h->grid_ritz = h->nsm * std::max(1, std::min(occ3, 2));
    CUDA_TRY(cudaFuncSetAttribute(k_correct<ST, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    CUDA_TRY(cudaFuncSetAttribute(k_restart_proj<ST, CT, kRitzKB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(1024 * kRitzKB * sizeof(double))));
    CUDA_TRY(cudaFuncSetAttribute(k_ritz<ST, CT, kRitzKB, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(1024 * kRitzKB * sizeof(double))));
    CUDA_TRY(cudaFuncSetAttribute(k_ritz<ST, CT, kRitzKB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(1024 * kRitzKB * sizeof(double))));
    if constexpr (std::is_same<CT, double>::value) {
        // fp64 tensor-core output pass when the coefficients fit 96 KB of shared memory
        const int tn = h->K <= 8 ? 1 : h->K <= 16 ? 2 : h->K <= 24 ? 3 : 4;
        const size_t smem = ((size_t)((h->m + 3) & ~3) * 8 * tn + 8 * tn) * sizeof(double);
        h->ritz_tn = (smem <= 96 * 1024 && h->ritz_mode != 1) ? tn : 0;
        for (auto f : {&k_ritz_mma<ST, 1>, &k_ritz_mma<ST, 2>, &k_ritz_mma<ST, 3>, &k_ritz_mma<ST, 4>})
            CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    }
}

static bool select_kernels(topk_eig_s *h) {
    using d = double;
    using f = float;
    if (h->ms == TOPK_F64 && h->vs == TOPK_F64 && h->cs == TOPK_F64) { set_kernels<d, d, d>(h); return true; }
    if (h->ms == TOPK_F32 && h->vs == TOPK_F32 && h->cs == TOPK_F64) { set_kernels<f, f, d>(h); return true; }
    if (h->ms == TOPK_F32 && h->vs == TOPK_F32 && h->cs == TOPK_F32) { set_kernels<f, f, f>(h); return true; }
    if (h->ms == TOPK_BF16 && h->vs == TOPK_F32 && h->cs == TOPK_F64) { set_kernels<bf16, f, d>(h); return true; }
    if (h->ms == TOPK_BF16 && h->vs == TOPK_BF16 && h->cs == TOPK_F64) { set_kernels<bf16, bf16, d>(h); return true; }
    return false;
}

// ---------------------------------------------------------------------------
static void carve_state(topk_eig_s *h, Part &p) {
    const int m = h->m, K = h->K;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 15) & ~size_t(15); return o; };
    size_t o_int = take(12 * sizeof(int));
    size_t o_ts = take(sizeof(double));
    size_t o_alpha = take((size_t)m * 8), o_beta = take((size_t)(m + 2) * 8), o_scale = take((size_t)(m + 1) * 8);
    size_t o_theta = take((size_t)m * 8), o_evals = take((size_t)K * 8), o_resid = take((size_t)K * 8);
    size_t o_coef = take((size_t)m * K * 8);
    p.state_bytes = off;
    p.state = h->alloc<char>(off);
    p.hstate.assign(off, 0);
    char *b = p.state;
    int *ints = reinterpret_cast<int *>(b + o_int);
    p.st.done = ints + 0;
    p.st.m_found = ints + 1;
    p.st.k_found = ints + 2;
    p.st.jac_sweeps = ints + 3;
    p.st.jac_conv = ints + 4;
    p.st.arrow_k = ints + 5;
    p.st.restarts = ints + 6;
    p.pro_gate = ints + 7;  // partial reorthogonalisation (reading Q29)
    p.pro_force = ints + 8;
    p.pro_count = ints + 9;
    if (h->reorth == 3) p.pro_w = h->alloc<double>((size_t)3 * (m + 2));
    p.st.tscale = reinterpret_cast<double *>(b + o_ts);
    p.st.alpha = reinterpret_cast<double *>(b + o_alpha);
    p.st.beta = reinterpret_cast<double *>(b + o_beta);
    p.st.scale = reinterpret_cast<double *>(b + o_scale);
    p.st.theta_all = reinterpret_cast<double *>(b + o_theta);
    p.st.evals = reinterpret_cast<double *>(b + o_evals);
    p.st.resid = reinterpret_cast<double *>(b + o_resid);
    p.st.coefS = reinterpret_cast<double *>(b + o_coef);
    p.st.tau = h->tau;
    // Gram matrix of the basis and the Ritz norms: device-only (not copied back per solve)
    p.st.gram = h->alloc<double>((size_t)m * m);
    p.st.rnrm2 = h->alloc<double>((size_t)K);
    p.st.m = m;
    p.st.use_gram = h->use_gram ? 1 : 0;
    // thick restart (reading Q26): arrowhead part of T and the kept Ritz coefficients
    p.st.keep = h->keep;
    p.st.arrow_theta = h->alloc<double>((size_t)std::max(h->keep, 1));
    p.st.arrow_b = h->alloc<double>((size_t)std::max(h->keep, 1));
    p.st.coefR = h->alloc<double>((size_t)m * std::max(h->keep, 1));
}

template <typename T> static T hget(const Part &p, const void *devptr) {
    T v;
    std::memcpy(&v, p.hstate.data() + ((const char *)devptr - p.state), sizeof(T));
    return v;
}
static const double *hptr(const Part &p, const double *devptr) {
    return reinterpret_cast<const double *>(p.hstate.data() + ((const char *)devptr - p.state));
}

// a4 on the device, in two halves:
//  upload_csr_slice: the part's canonical CSR slice goes up as is (row pointers rebased,
//    values rounded to the value storage dtype on the way, RNE straight from f64,
//    reading Q22, chunk by chunk into the pinned staging buffers, mem_pool.h). It
//    needs only the partition, so create runs it on a helper thread while the host
//    builds the degree order and the layout tables.
//  device_layout: k_layout_big / k_layout_sell scatter the slice into the physical
//    SpMV arrays with the rule of build_part.
struct DevCsr {
    int64_t *srp = nullptr;
    int32_t *scol = nullptr;
    void *sval = nullptr;
};
static void *dalloc_or_throw(size_t bytes) {
    void *q = pool_dev_alloc(std::max<size_t>(bytes, 256));
    if (!q) CUDA_TRY(cudaErrorMemoryAllocation);
    return q;
}
// nthreads: OpenMP threads of the fills, read before every 32 MB chunk (the creating
// thread raises it once its own host work is done)
static void upload_csr_slice(const Csr &csr, int64_t r0, int64_t ng, topk_dtype_t ms, DevCsr &d, cudaStream_t st,
                             const std::atomic<int> &nthreads) {
    const int64_t z0 = csr.rowptr[(size_t)r0], z = csr.rowptr[(size_t)(r0 + ng)] - z0;
    const size_t es = dsize(ms);
    d.srp = static_cast<int64_t *>(dalloc_or_throw((size_t)(ng + 1) * 8));
    d.scol = static_cast<int32_t *>(dalloc_or_throw((size_t)z * 4));
    d.sval = dalloc_or_throw((size_t)z * es);
    const int64_t *srp = csr.rowptr.data() + r0;
    auto fill_srp = [&](char *dst, size_t off, size_t nb) {
        omp_set_num_threads(nthreads.load());
        const size_t i0 = off / 8, cnt = nb / 8;
        int64_t *dd = reinterpret_cast<int64_t *>(dst);
#pragma omp parallel for schedule(static)
        for (size_t i = 0; i < cnt; ++i) dd[i] = srp[i0 + i] - z0;
    };
    CUDA_TRY(staged_h2d(d.srp, (size_t)(ng + 1) * 8, fill_srp, st));
    const char *sc = reinterpret_cast<const char *>(csr.col.data() + z0);
    CUDA_TRY(staged_h2d(d.scol, (size_t)z * 4, [&](char *dst, size_t off, size_t nb) {
        omp_set_num_threads(nthreads.load());
        par_memcpy(dst, sc + off, nb);
    }, st));
    const double *sv = csr.val.data() + z0;
    auto fill_val = [&](char *dst, size_t off, size_t nb) {
        omp_set_num_threads(nthreads.load());
        const size_t k0 = off / es, cnt = nb / es;
#pragma omp parallel for schedule(static)
        for (size_t k = 0; k < cnt; ++k) {
            const double x = sv[k0 + k];
            if (ms == TOPK_F64) reinterpret_cast<double *>(dst)[k] = x;
            else if (ms == TOPK_F32) reinterpret_cast<float *>(dst)[k] = round_f32(x);
            else reinterpret_cast<uint16_t *>(dst)[k] = round_bf16_bits(x);
        }
    };
    CUDA_TRY(staged_h2d(d.sval, (size_t)z * es, fill_val, st));
}
static void free_dev_csr(DevCsr &d) {
    pool_dev_free(d.srp);
    pool_dev_free(d.scol);
    pool_dev_free(d.sval);
    d = DevCsr{};
}
// Device arrays and work tables of one SpMV pass (tables uploaded here).
static void alloc_pass(topk_eig_s *h, SpmvDev &d, const std::vector<Chunk> &chunks, const std::vector<LongRow> &longrows,
                       const std::vector<int64_t> &sell, const std::vector<int32_t> &items, const std::vector<int64_t> &bigptr,
                       int64_t nphys, size_t val_es) {
    d.nchunks = (int)chunks.size();
    d.nlong = (int)longrows.size();
    d.nitems = (int)items.size() / 2;
    d.nphys = nphys;
    d.col = h->alloc<int32_t>((size_t)nphys + 128);  // physical col/val padded by 128 entries
    d.val = h->alloc<char>(((size_t)nphys + 128) * val_es);
    d.chunks = h->alloc<Chunk>(chunks.size());
    d.longrows = h->alloc<LongRow>(longrows.size());
    d.sell = h->alloc<int64_t>(sell.size());
    d.items = h->alloc<int32_t>(items.size());
    d.long_parts = h->alloc<double>(chunks.size());
    d.long_cnt = h->alloc<unsigned>(longrows.size());
    d.alpha_long = h->alloc<double>(longrows.size());
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (!chunks.empty()) CUDA_TRY(scopy(h->stream, d.chunks, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
    if (!longrows.empty()) CUDA_TRY(scopy(h->stream, d.longrows, longrows.data(), longrows.size() * sizeof(LongRow), cudaMemcpyHostToDevice));
    if (!sell.empty()) CUDA_TRY(scopy(h->stream, d.sell, sell.data(), sell.size() * 8, cudaMemcpyHostToDevice));
    if (!items.empty()) CUDA_TRY(scopy(h->stream, d.items, items.data(), items.size() * 4, cudaMemcpyHostToDevice));
    d.h_sell = sell;
    d.h_bigptr = bigptr;
}

template <typename VT, int MODE>
static void scatter_pass(topk_eig_s *h, Part &p, const PartLayout &L, const DevCsr &d, const int32_t *d_colmap,
                         const int64_t *d_drp, SpmvDev &dp) {
    const VT *sval = static_cast<const VT *>(d.sval);
    if (L.nbig > 0 && MODE == 0) {
        if (dp.nchunks > 0) {
            k_layout_big_chunks<VT><<<h->nsm * 8, 256, 0, h->stream>>>(d.srp, d.scol, sval, p.perm, d_drp, dp.chunks, dp.nchunks,
                                                                       d_colmap, dp.nphys, dp.col, reinterpret_cast<VT *>(dp.val));
            CUDA_TRY(cudaGetLastError());
        }
    } else if (L.nbig > 0) {
        int64_t *d_big = static_cast<int64_t *>(dalloc_or_throw(dp.h_bigptr.size() * 8));
        CUDA_TRY(scopy(h->stream, d_big, dp.h_bigptr.data(), dp.h_bigptr.size() * 8, cudaMemcpyHostToDevice));
        k_layout_big<VT, MODE><<<h->nsm * 8, 256, 0, h->stream>>>(d.srp, d.scol, sval, p.perm, d_big, d_colmap, L.nbig,
                                                                 dp.nphys, p.npad, p.g, dp.col, reinterpret_cast<VT *>(dp.val));
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        pool_dev_free(d_big);
    }
    const int64_t nsl = (int64_t)dp.h_sell.size() / 2;
    if (nsl > 0) {
        k_layout_sell<VT, MODE><<<h->nsm * 8, 256, 0, h->stream>>>(d.srp, d.scol, sval, p.perm, d_drp, d_colmap,
                                                                  reinterpret_cast<const longlong2 *>(dp.sell), (int64_t)L.nbig,
                                                                  L.nnonempty, nsl, dp.nphys, p.npad, p.g, dp.col,
                                                                  reinterpret_cast<VT *>(dp.val));
        CUDA_TRY(cudaGetLastError());
    }
}

// a4, second half: the SpMV passes of part p from its uploaded CSR slice with the rule of
// build_part. Two-pass SpMV (h->split): the own-slot entries per position are counted on
// the device, both passes' tables built on the host (build_pass_tables), and the entries
// scattered into the own-slot pass and the final pass.
template <typename VT>
static void device_layout_t(topk_eig_s *h, Part &p, const PartLayout &L, const DevCsr &d, const int32_t *d_colmap) {
    const int64_t ng = L.nrows;
    int64_t *d_drp = static_cast<int64_t *>(dalloc_or_throw((size_t)(ng + 1) * 8));
    const char *drp = reinterpret_cast<const char *>(L.rowptr.data());
    CUDA_TRY(staged_h2d(d_drp, (size_t)(ng + 1) * 8, [&](char *dst, size_t off, size_t nb) { par_memcpy(dst, drp + off, nb); },
                        h->stream));
    if (!h->split) {
        const std::vector<int64_t> bigptr(L.rowptr.begin(), L.rowptr.begin() + L.nbig + 1);
        alloc_pass(h, p.sp, L.chunks, L.longrows, L.sell, L.items, bigptr, L.nphys, sizeof(VT));
        scatter_pass<VT, 0>(h, p, L, d, d_colmap, d_drp, p.sp);
    } else {
        const int64_t nne = L.nnonempty;
        p.owndeg = h->alloc<int32_t>((size_t)std::max<int64_t>(nne, 1));
        if (nne > 0) {
            k_own_count<<<h->nsm * 8, 256, 0, h->stream>>>(d.srp, d.scol, p.perm, d_colmap, nne, p.npad, p.g, p.owndeg);
            CUDA_TRY(cudaGetLastError());
        }
        std::vector<int32_t> od((size_t)std::max<int64_t>(ng, 1), 0), rd((size_t)std::max<int64_t>(ng, 1), 0);
        if (nne > 0) CUDA_TRY(scopy(h->stream, od.data(), p.owndeg, (size_t)nne * 4, cudaMemcpyDeviceToHost));
        for (int64_t q = 0; q < ng; ++q) rd[(size_t)q] = (int32_t)(L.rowptr[(size_t)q + 1] - L.rowptr[(size_t)q]) - od[(size_t)q];
        PassTables To, Tr;
        build_pass_tables(od.data(), L.nbig, nne, false, To);
        build_pass_tables(rd.data(), L.nbig, nne, true, Tr);
        alloc_pass(h, p.own, To.chunks, To.longrows, To.sell, To.items, To.bigptr, To.nphys, sizeof(VT));
        alloc_pass(h, p.sp, Tr.chunks, Tr.longrows, Tr.sell, Tr.items, Tr.bigptr, Tr.nphys, sizeof(VT));
        p.ypart = h->alloc<double>((size_t)std::max<int64_t>(p.npad, 1));  // rows without own entries stay 0
        scatter_pass<VT, 1>(h, p, L, d, d_colmap, d_drp, p.own);
        scatter_pass<VT, 2>(h, p, L, d, d_colmap, d_drp, p.sp);
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    pool_dev_free(d_drp);
}
static void device_layout(topk_eig_s *h, Part &p, const PartLayout &L, const DevCsr &d, const int32_t *d_colmap) {
    if (h->ms == TOPK_F64) device_layout_t<double>(h, p, L, d, d_colmap);
    else if (h->ms == TOPK_F32) device_layout_t<float>(h, p, L, d, d_colmap);
    else device_layout_t<uint16_t>(h, p, L, d, d_colmap);
}

static int64_t model_bytes(topk_eig_s *h, const Part &p) {
    // B_spmv = z(4+s_v) + 4(n_g+1) + s n_x + s n_g; B_step(i) = (2i+4) n_g s;
    // Ritz: (m + 3K) n_g s. Per part, whole solve.
    const int64_t s = (int64_t)dsize(h->vs), sv = (int64_t)dsize(h->ms);
    const int64_t nx = (h->G == 1) ? p.nrows : h->n;
    int64_t b = 0;
    for (int i = 1; i <= h->m; ++i) {
        b += p.nnz * (4 + sv) + 4 * (p.nrows + 1) + s * nx + s * p.nrows;
        const bool ro = h->reorth > 0 && (h->period <= 1 || i % h->period == 0 || (i > 1 && (i - 1) % h->period == 0));
        b += ro ? (2 * i + 4) * p.nrows * s : 4 * p.nrows * s;
    }
    b += (int64_t)(h->m + 3 * h->K) * p.nrows * s;
    return b;
}

// halo set-up for part p (reading Q27): compact column map, remote-entry lists, and
// with one process per GPU the request lists exchanged so every rank knows which of
// its positions each peer needs
static void setup_halo(topk_eig_s *h, Part &p, const Csr &csr, int64_t npad, const int32_t *pos, int32_t *d_colmap) {
    Halo H;
    build_halo(csr, h->bounds.data(), h->G, p.g, npad, pos, H);
    const char *cm = reinterpret_cast<const char *>(H.colmap.data());
    CUDA_TRY(staged_h2d(d_colmap, H.colmap.size() * 4, [&](char *dst, size_t off, size_t nb) { par_memcpy(dst, cm + off, nb); },
                        h->stream));
    p.nhalo = H.n;
    p.halo_off = H.off;
    p.halo_pos_h = H.pos;
    std::vector<int32_t> hq((size_t)H.n);
    for (int q = 0; q < h->G; ++q)
        for (int64_t t = H.off[(size_t)q]; t < H.off[(size_t)q + 1]; ++t) hq[(size_t)t] = q;
    p.halo_q = h->alloc<int32_t>((size_t)std::max<int64_t>(H.n, 1));
    p.halo_pos = h->alloc<int32_t>((size_t)std::max<int64_t>(H.n, 1));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (H.n) {
        CUDA_TRY(scopy(h->stream, p.halo_q, hq.data(), (size_t)H.n * 4, cudaMemcpyHostToDevice));
        CUDA_TRY(scopy(h->stream, p.halo_pos, H.pos.data(), (size_t)H.n * 4, cudaMemcpyHostToDevice));
    }
    if (!h->comm) return;
    // counts[r][q] = entries rank r receives from q; rank g sends counts[q][g] to q
    const int G = h->G, g = h->rank;
    int64_t *d_cnt = h->alloc<int64_t>((size_t)G * G);
    std::vector<int64_t> mine((size_t)G);
    for (int q = 0; q < G; ++q) mine[(size_t)q] = H.off[(size_t)q + 1] - H.off[(size_t)q];
    CUDA_TRY(scopy(h->stream, d_cnt + (size_t)g * G, mine.data(), (size_t)G * 8, cudaMemcpyHostToDevice));
    NCCL_TRY(ncclAllGather(d_cnt + (size_t)g * G, d_cnt, (size_t)G, ncclInt64, h->comm, h->stream));
    std::vector<int64_t> cnt((size_t)G * G);
    CUDA_TRY(cudaMemcpyAsync(cnt.data(), d_cnt, cnt.size() * 8, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    p.send_off.assign((size_t)G + 1, 0);
    for (int q = 0; q < G; ++q) p.send_off[(size_t)q + 1] = p.send_off[(size_t)q] + (q == g ? 0 : cnt[(size_t)q * G + g]);
    const int64_t nsend = p.send_off[(size_t)G];
    p.send_pos = h->alloc<int32_t>((size_t)std::max<int64_t>(nsend, 1));
    p.sendbuf = h->alloc<char>((size_t)std::max<int64_t>(nsend, 1) * dsize(h->vs));
    NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < G; ++q) {
        if (q == g) continue;
        const size_t nr = (size_t)(H.off[(size_t)q + 1] - H.off[(size_t)q]);  // I request from q
        const size_t ns = (size_t)(p.send_off[(size_t)q + 1] - p.send_off[(size_t)q]);  // q requests from me
        if (nr) NCCL_TRY(ncclSend(p.halo_pos + H.off[(size_t)q], nr, ncclInt32, q, h->comm, h->stream));
        if (ns) NCCL_TRY(ncclRecv(p.send_pos + p.send_off[(size_t)q], ns, ncclInt32, q, h->comm, h->stream));
    }
    NCCL_TRY(ncclGroupEnd());
    CUDA_TRY(cudaStreamSynchronize(h->stream));
}

static topk_status_t create_impl(topk_eig_t *out, const topk_matrix_t *A, int32_t K,
                                 topk_dtype_t storage, topk_dtype_t compute,
                                 const topk_eig_opts_t *opts) {
    if (!out || !A) return fail(TOPK_E_INVALID, "out and A must be non-NULL");
    *out = nullptr;
    topk_eig_opts_t o{};
    if (opts) std::memcpy(&o, opts, std::min<size_t>(sizeof(o), opts->struct_size ? opts->struct_size : sizeof(o)));
    const int64_t n = A->n;
    if (n < 1 || n >= (1ll << 31)) return fail(TOPK_E_INVALID, "n must be in [1, 2^31)");
    const int m = o.krylov_dim > 0 ? o.krylov_dim : K;
    if (K < 1 || K > n || K > 256) return fail(TOPK_E_INVALID, "K must be in [1, min(n, 256)]");
    if (m < K || m > n || m > 1024) return fail(TOPK_E_INVALID, "krylov_dim must be in [K, min(n, 1024)]");
    const int world = o.world > 1 ? o.world : 1;
    const int G = o.num_parts > 0 ? o.num_parts : world;
    if (world > 1 && (G != world || o.rank < 0 || o.rank >= world || !o.nccl_id))
        return fail(TOPK_E_INVALID, "multi-process: num_parts must equal world, 0 <= rank < world, nccl_id non-NULL");
    if (G < 1 || G > 64 || G > n) return fail(TOPK_E_INVALID, "num_parts must be in [1, min(n, 64)]");
    topk_dtype_t ms = (o.values_storage > 0) ? (topk_dtype_t)o.values_storage : storage;
    if (storage < TOPK_F64 || storage > TOPK_BF16 || compute < TOPK_F64 || compute > TOPK_F32 || ms < TOPK_F64 || ms > TOPK_BF16)
        return fail(TOPK_E_INVALID, "bad dtype");

    {  // the (values, vectors, compute) combinations select_kernels instantiates
        const bool ok = (ms == TOPK_F64 && storage == TOPK_F64 && compute == TOPK_F64) ||
                        (ms == TOPK_F32 && storage == TOPK_F32) ||
                        (ms == TOPK_BF16 && storage == TOPK_F32 && compute == TOPK_F64) ||
                        (ms == TOPK_BF16 && storage == TOPK_BF16 && compute == TOPK_F64);
        if (!ok) return fail(TOPK_E_INVALID, "unsupported (values, storage, compute) dtype combination");
    }
    std::unique_ptr<topk_eig_s> h(new topk_eig_s());
    h->n = n; h->K = K; h->m = m; h->G = G; h->world = world; h->rank = world > 1 ? o.rank : 0;
    h->vs = storage; h->ms = ms; h->cs = compute;
    h->reorth = o.reorth == 0 ? 1 : o.reorth;
    if (h->reorth != 1 && h->reorth != 2 && h->reorth != 3 && h->reorth != -1)
        return fail(TOPK_E_INVALID, "reorth must be 1, 2, 3 or -1");
    h->tau = o.breakdown_tol > 0 ? o.breakdown_tol : (storage == TOPK_F64 ? 1e-12 : storage == TOPK_F32 ? 1e-6 : 1e-3);
    if (compute == TOPK_F32 && storage == TOPK_F64) return fail(TOPK_E_INVALID, "compute must be at least as precise as storage");
    if (!(o.conv_tol >= 0.0) || o.conv_check < 0) return fail(TOPK_E_INVALID, "conv_tol must be >= 0 and conv_check >= 0");
    h->conv_tol = o.conv_tol;
    if (o.reorth_period < 0) return fail(TOPK_E_INVALID, "reorth_period must be >= 0");
    h->period = o.reorth_period > 1 ? o.reorth_period : 1;
    if (h->period > 1 && h->reorth != 1) return fail(TOPK_E_INVALID, "reorth_period > 1 needs reorth = 1");
    if (h->period > 1 && o.restart_keep > 0) return fail(TOPK_E_INVALID, "thick restart needs reorthogonalisation every iteration");
    if (o.restart_keep < 0 || o.max_restarts < 0) return fail(TOPK_E_INVALID, "restart_keep and max_restarts must be >= 0");
    if (o.restart_keep > 0) {
        if (o.restart_keep < K || o.restart_keep > m - 2 || o.restart_keep > 256)
            return fail(TOPK_E_INVALID, "restart_keep must be in [K, min(krylov_dim - 2, 256)]");
        if (h->reorth < 0 || h->reorth == 3) return fail(TOPK_E_INVALID, "thick restart needs full reorthogonalisation (reorth 1 or 2)");
        h->keep = o.restart_keep;
        h->max_restarts = o.max_restarts;
    }
    h->conv_check = o.conv_check > 0 ? o.conv_check : K;
    if (h->conv_tol > 0.0 && h->period > 1)
        return fail(TOPK_E_INVALID, "conv_tol > 0 is not supported with reorth_period > 1");
    if (h->conv_tol > 0.0 && h->keep == 0)  // the checks enqueued per solve (thick restart tests per cycle)
        for (int i = K; i < m; ++i) h->conv_checks += (i % h->conv_check == 0);
    if (o.exchange < 0 || o.exchange > 1) return fail(TOPK_E_INVALID, "exchange must be 0 (allgather) or 1 (halo)");
    h->halo = (G > 1 && o.exchange == 1);
    if (o.overlap < -1 || o.overlap > 1) return fail(TOPK_E_INVALID, "overlap must be -1, 0 or 1");
    // two-pass SpMV, own-slot columns first: overlap = 1 always (also in
    // one process); by default (0) with one process per GPU when the vector exchange is large
    // enough to pay for the second pass (measured at G = 8: +31 us per SpMV at C3, whose
    // exchange is ~15 MB; +45 us at C4, ~350 MB; profiles/r02_overlap_cost.jsonl), decided
    // below once n_pad is known
    h->split = G > 1 && !h->halo && o.overlap == 1;
    if (o.jacobi_path < 0 || o.jacobi_path > 2) return fail(TOPK_E_INVALID, "jacobi_path must be 0, 1 or 2");
    if (o.jacobi_cluster != 0 && o.jacobi_cluster != 8 && o.jacobi_cluster != 16)
        return fail(TOPK_E_INVALID, "jacobi_cluster must be 0, 8 or 16");
    h->restart_unrolled = o.restart_loop == 1;
    if (o.ritz_path < 0 || o.ritz_path > 1) return fail(TOPK_E_INVALID, "ritz_path must be 0 or 1");
    h->ritz_mode = o.ritz_path;
    h->use_graph = o.use_graph >= 0;
    h->profile = o.profile > 0;
    h->device = o.device;

    // a1-a3 on the host
    Csr csr;
    std::string err;
    StageClock clk;
    topk_status_t s = canonicalize(*A, csr, err);
    if (s != TOPK_OK) return fail(s, err);
    clk.mark("canonicalize");
    // one process: the whole matrix here; one process per GPU: each rank hashes its own
    // rows and the sums are added over the ranks once the communicator exists (below)
    if (world == 1 && o.check_symmetry >= 0 && !is_symmetric(csr))
        return fail(TOPK_E_NOT_SYMMETRIC, "matrix is not symmetric");
    clk.mark("symmetry check");
    h->bounds.resize((size_t)G + 1);
    s = partition_rule_p(csr.rowptr.data(), n, G, h->bounds.data());
    if (s != TOPK_OK) return fail(s, "partition failed");
    const int64_t npad = padded_rows(h->bounds.data(), G);
    clk.mark("partition");
    if (G > 1 && !h->halo && o.overlap == 0 && world > 1)  // >= 64 MB received per exchange
        h->split = (int64_t)(G - 1) * npad * (int64_t)dsize(storage) >= ((int64_t)64 << 20);

    // device
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(TOPK_E_NODEVICE, "no CUDA device: this library runs only on sm_100 (B200); there is no CPU fallback");
    if (h->device < 0 || h->device >= ndev) return fail(TOPK_E_INVALID, "bad device ordinal");
    try {
        CUDA_TRY(cudaSetDevice(h->device));
        int major = 0, minor = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, h->device));
        CUDA_TRY(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, h->device));
        if (major != 10 || minor != 0)
            return fail(TOPK_E_NODEVICE, "device is not sm_100 (B200); this library is built for sm_100a only");
        CUDA_TRY(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->device));
        CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreate(&h->ev0));
        CUDA_TRY(cudaEventCreate(&h->ev1));
        CUDA_TRY(cudaEventCreate(&h->evL));
        if (h->split && world > 1) {
            CUDA_TRY(cudaStreamCreateWithFlags(&h->comm_stream, cudaStreamNonBlocking));
            CUDA_TRY(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        }
        CUDA_TRY(cudaEventCreate(&h->evJ));
        clk.mark("device init");
        // a4, first half, in the background: the local parts' CSR slices go up on a
        // helper thread (own stream) while this thread builds the degree order and tables
        const int nloc = (world > 1) ? 1 : G;
        std::vector<DevCsr> dcsr((size_t)nloc);
        std::string up_err;
        // the host cores are split between the uploader and this thread while both run
        // (two full OpenMP teams oversubscribe the cores: C3 create 57-60 ms with both at
        // all cores, 49-50 ms split in halves, 71-78 ms with a quarter for the upload)
        const int omp_all = omp_get_max_threads();
        const int omp_half = std::max(1, omp_all / 2);
        struct OmpRestore {
            int n;
            ~OmpRestore() { omp_set_num_threads(n); }
        } omp_restore{omp_all};
        std::atomic<int> up_threads{omp_half};
        std::thread uploader([&] {
            cudaStream_t st = nullptr;
            try {
                CUDA_TRY(cudaSetDevice(h->device));
                CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
                for (int lp = 0; lp < nloc; ++lp) {
                    const int g = (world > 1) ? h->rank : lp;
                    upload_csr_slice(csr, h->bounds[(size_t)g], h->bounds[(size_t)g + 1] - h->bounds[(size_t)g], ms,
                                     dcsr[(size_t)lp], st, up_threads);
                }
            } catch (CudaFail &e) {
                up_err = e.msg;
            } catch (std::bad_alloc &) {
                up_err = "host allocation failed";
            }
            if (st) cudaStreamDestroy(st);
        });
        struct Joiner {
            std::thread &t;
            std::vector<DevCsr> &d;
            ~Joiner() {
                if (t.joinable()) t.join();
                for (DevCsr &x : d) free_dev_csr(x);
            }
        } joiner{uploader, dcsr};
        omp_set_num_threads(std::max(1, omp_all - omp_half));
        hvec<int32_t> pos;
        degree_order(csr, h->bounds.data(), G, pos);
        const hvec<int32_t> colmap = column_map(n, h->bounds.data(), G, npad, pos.data());
        clk.mark("degree order + column map");
        if (!select_kernels(h.get())) return fail(TOPK_E_INVALID, "unsupported (values, storage, compute) dtype combination");
        clk.mark("kernel attributes");

        // exchange buffers (shared by the local parts)
        h->ex.alpha_part = h->alloc<double>((size_t)G);
        h->ex.norm_part = h->alloc<double>((size_t)G);
        h->ex.hpart = h->alloc<double>((size_t)G * 2 * (m + 1));
        h->ex.ritz_part = h->alloc<double>((size_t)G * K);
        h->ex.rst_part = h->alloc<double>((size_t)G * std::max(h->keep, 1));

        if (G > 1 && !h->halo) h->replica = h->alloc<char>((size_t)G * npad * dsize(storage));
        h->ex.replica = h->replica;
        const int nlocal = (world > 1) ? 1 : G;
        h->dparams = h->alloc<SolveParams>(1 + (size_t)nlocal);
        h->hparams_own.assign((size_t)(1 + nlocal), SolveParams{});
        h->hparams = h->hparams_own.data();
        // Jacobi workspace: T and S with a power-of-two leading dimension, + rotations
        const int M = m + (m & 1);
        int ls = 0, hs = 0;
        while ((1 << ls) < M) ++ls;
        while ((1 << hs) < M / 2) ++hs;
        h->jac_ld_log2 = ls;
        h->jac_hl_log2 = hs;
        const size_t jbytes = (size_t)2 * M * ((size_t)1 << ls) * 8 + (size_t)M * 8 + (size_t)M * 4 + (size_t)M * 2 + 64;
        const int items = std::max((M / 2) << hs, (M / 2) << ls);
        // one thread per 2x2 block update / S column pair of a round (measured: a
        // single warp serialising them is 3x slower at m = 24)
        h->jac_threads = std::max(32, std::min(1024, (items + 31) / 32 * 32));
        {
            cudaFuncAttributes fa{};
            CUDA_TRY(cudaFuncGetAttributes(&fa, k_jacobi<false>));
            h->jac_threads = std::min(h->jac_threads, fa.maxThreadsPerBlock / 32 * 32);
            CUDA_TRY(cudaFuncGetAttributes(&fa, k_jacobi<true>));
            h->jac_threads = std::min(h->jac_threads, fa.maxThreadsPerBlock / 32 * 32);
#ifdef TOPK_JAC_THREADS  // dev build variant (A/B of the CTA size)
            h->jac_threads = std::max(32, std::min(h->jac_threads, TOPK_JAC_THREADS / 32 * 32));
#endif
        }
        // single CTA in shared memory for M <= 40; above that the cluster path is
        // faster (tools/jac_timing.py, profiles/r01_jacobi_timing.jsonl: m = 48 1.06 vs
        // 1.27 ms, m = 96 2.7 vs 8.4 ms, m = 192 10.9 vs 106 ms)
        // opts.jacobi_path: 0 auto (as above), 1 single CTA only (shared memory up to
        // M = 40, global memory above), 2 cluster at any m
        if (jbytes <= 200 * 1024 && M <= 40 && o.jacobi_path != 2) {
            h->jac_smem = jbytes;
            CUDA_TRY(cudaFuncSetAttribute(k_jacobi<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jbytes));
        } else {
            h->jac_smem = 0;
            h->jac_bytes = (jbytes + 255) / 256 * 256;
            h->jac_work = h->alloc<double>((size_t)nlocal * h->jac_bytes / 8);
            // T, S distributed over a thread-block cluster when they fit its shared memory
            const int first = o.jacobi_cluster ? o.jacobi_cluster : (M >= 96 ? 16 : 8);
            for (int CL : {first, 24 - first}) {
                if (o.jacobi_path == 1) break;
                const size_t R = (size_t)(M + CL - 1) / CL;
                const size_t cb = 3 * R * M * 8 + (size_t)M * 8 + (size_t)(2 * M + M) * 4 + 64;
                if (cb > 200 * 1024) continue;
                CUDA_TRY(cudaFuncSetAttribute(k_jacobi_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cb));
                if (CL > 8) CUDA_TRY(cudaFuncSetAttribute(k_jacobi_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)CL);
                cfg.blockDim = dim3(kJacClNT);
                cfg.dynamicSmemBytes = cb;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = (unsigned)CL;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                int ncl = 0;
                if (cudaOccupancyMaxActiveClusters(&ncl, k_jacobi_cl, &cfg) != cudaSuccess || ncl < 1) {
                    cudaGetLastError();
                    continue;
                }
                h->jac_cl = CL;
                h->jac_cl_smem = cb;
                break;
            }
        }

        if (world > 1) {  // before the parts: the halo set-up exchanges request lists
            ncclUniqueId id;
            std::memcpy(&id, o.nccl_id, sizeof(id));
            NCCL_TRY(ncclCommInitRank(&h->comm, world, id, h->rank));
            if (o.check_symmetry >= 0) {  // a2, distributed: the multiset hash sums are additive
                uint64_t hs[4];
                symmetry_sums(csr, h->bounds[(size_t)h->rank], h->bounds[(size_t)h->rank + 1], hs);
                uint64_t *d_hs = h->alloc<uint64_t>(4);
                CUDA_TRY(scopy(h->stream, d_hs, hs, sizeof(hs), cudaMemcpyHostToDevice));
                NCCL_TRY(ncclAllReduce(d_hs, d_hs, 4, ncclUint64, ncclSum, h->comm, h->stream));
                CUDA_TRY(scopy(h->stream, hs, d_hs, sizeof(hs), cudaMemcpyDeviceToHost));
                if (!(hs[0] == hs[2] && hs[1] == hs[3])) return fail(TOPK_E_NOT_SYMMETRIC, "matrix is not symmetric");
            }
        }
        // column map (global column -> device column entry), shared by the local parts
        // (with the halo exchange each part uploads its own compact map instead)
        int32_t *d_colmap = static_cast<int32_t *>(pool_dev_alloc((size_t)n * 4));
        if (!d_colmap) CUDA_TRY(cudaErrorMemoryAllocation);
        struct ColmapGuard { int32_t *p; ~ColmapGuard() { pool_dev_free(p); } } colmap_guard{d_colmap};
        h->parts.resize((size_t)nlocal);
        for (int lp = 0; lp < nlocal; ++lp) {
            Part &p = h->parts[(size_t)lp];
            p.g = (world > 1) ? h->rank : lp;
            PartLayout L;
            s = build_part_tables(csr, h->bounds.data(), G, p.g, npad, pos.data(), L, err);
            if (s != TOPK_OK) return fail(s, err);
            clk.mark("layout tables");
            p.row0 = L.row0; p.nrows = L.nrows; p.npad = npad; p.nnz = (int64_t)L.rowptr.back();
            p.nbig = L.nbig; p.nnonempty = L.nnonempty;
            p.perm = h->alloc<int32_t>(L.perm.size());
            p.inv = h->alloc<int32_t>(L.perm.size());
            CUDA_TRY(cudaStreamSynchronize(h->stream));
            if (!L.perm.empty()) {
                hvec<int32_t> inv(L.perm.size());
#pragma omp parallel for schedule(static)
                for (size_t q = 0; q < L.perm.size(); ++q) inv[(size_t)L.perm[q]] = (int32_t)q;
                CUDA_TRY(scopy(h->stream, p.perm, L.perm.data(), L.perm.size() * 4, cudaMemcpyHostToDevice));
                CUDA_TRY(scopy(h->stream, p.inv, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
            }
            if (h->halo) setup_halo(h.get(), p, csr, npad, pos.data(), d_colmap);
            if (lp + 1 == nlocal) up_threads.store(omp_all);  // this thread's host work is done: the upload takes every core
            if (lp == 0 && !h->halo) {  // after the first part's tables: the staging buffers are the uploader's until then
                const char *cm = reinterpret_cast<const char *>(colmap.data());
                CUDA_TRY(staged_h2d(d_colmap, (size_t)n * 4, [&](char *dst, size_t off, size_t nb) { par_memcpy(dst, cm + off, nb); },
                                    h->stream));
            }
            if (uploader.joinable()) {
                uploader.join();
                omp_set_num_threads(omp_all);
                clk.mark("wait for CSR upload");
                if (!up_err.empty()) throw CudaFail(up_err);
            }
            device_layout(h.get(), p, L, dcsr[(size_t)lp], d_colmap);
            free_dev_csr(dcsr[(size_t)lp]);
            p.h_rowptr = std::move(L.rowptr);  // host copies for the exports
            p.h_perm = std::move(L.perm);
            clk.mark("device layout");
            const size_t vsz = dsize(storage);
            p.V = h->alloc<char>((size_t)(m + 1) * npad * vsz);
            p.y = h->alloc<char>((size_t)npad * vsz);
            p.w = h->alloc<char>((size_t)npad * vsz);
            if (h->keep > 0) p.Vs = h->alloc<char>((size_t)h->keep * npad * vsz);
            if (h->halo) p.xg = h->alloc<char>((size_t)(npad + p.nhalo) * vsz);
            p.out = h->alloc<double>((size_t)K * std::max<int64_t>(p.nrows, 1));
            p.yt = h->alloc<double>((size_t)((K + kRitzKB - 1) / kRitzKB) * kRitzKB * std::max<int64_t>(p.npad, 1));
            p.v1buf = h->alloc<double>((size_t)std::max<int64_t>(p.nrows, 1));
            p.slots = h->alloc<double>((size_t)std::max(std::max(h->grid_spmv, h->grid_corr), std::max(std::max(h->grid_stream, h->grid_step), h->grid_ritz)) * (size_t)std::max(2 * (m + 2), K) + 64);
            p.counters = h->alloc<unsigned>(8 + 64);
            carve_state(h.get(), p);
            h->bytes_model += model_bytes(h.get(), p);
            clk.mark("allocations");
        }
        if (h->comm) {  // interconnect bytes received per solve (model, fixed m: v1 + one exchange per step)
            const int64_t es = (int64_t)dsize(storage);
            const int64_t vec = h->halo ? h->parts[0].nhalo * es : (int64_t)(G - 1) * npad * es;
            const int64_t scal = (int64_t)(G - 1) * 8 * (3 + 2 * (m + 1));  // alpha, norm, [h, Gram] per step
            h->bytes_nvlink = (int64_t)(m + 1) * vec + (int64_t)m * scal + (int64_t)(G - 1) * 8 * K;
        }
        if (h->halo && !h->comm) {  // parts on one device pull from each other's x_g
            std::vector<const void *> src;
            for (Part &p : h->parts) src.push_back(p.xg);
            h->d_xsrc = h->alloc<const void *>(src.size());
            CUDA_TRY(scopy(h->stream, h->d_xsrc, src.data(), src.size() * sizeof(void *), cudaMemcpyHostToDevice));
        }
        CUDA_TRY(cudaStreamSynchronize(h->stream));
    } catch (CudaFail &e) {
        return fail(TOPK_E_CUDA, e.msg);
    } catch (NcclFail &e) {
        return fail(TOPK_E_NCCL, e.msg);
    } catch (std::bad_alloc &) {
        return fail(TOPK_E_NOMEM, "host allocation failed");
    }
    *out = h.release();
    return TOPK_OK;
}

topk_eig_s::~topk_eig_s() {
    StageClock clk;
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    clk.mark("destroy: stream sync");
    if (gexec) cudaGraphExecDestroy(gexec);
    clk.mark("destroy: graph");
    if (comm) ncclCommDestroy(comm);
    for (void *p : allocs) pool_dev_free(p);  // back to the cache (the stream is idle)
    clk.mark("destroy: pool");
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (evL) cudaEventDestroy(evL);
    if (evJ) cudaEventDestroy(evJ);
    for (auto &q : prof) { cudaEventDestroy(q.a); cudaEventDestroy(q.b); }
    clk.mark("destroy: events");
    if (stream) cudaStreamDestroy(stream);
    if (body_stream) cudaStreamDestroy(body_stream);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    clk.mark("destroy: stream");
}

static void free_handle(topk_eig_s *h) { delete h; }

// Enqueue one full solve on h->stream (graph replay or eager launches).
static void enqueue(topk_eig_s *h, uint64_t seed, const double *v1_host, void *const *out_ptrs, int out_dtype) {
    const int nl = (int)h->parts.size();
    h->hparams[0].seed = seed;
    h->hparams[0].use_v1 = v1_host ? 1 : 0;
    h->hparams[0].out_dtype = out_dtype;
    for (int lp = 0; lp < nl; ++lp) h->hparams[1 + lp].out_ptr = out_ptrs ? out_ptrs[lp] : nullptr;
    CUDA_TRY(cudaMemcpyAsync(h->dparams, h->hparams, sizeof(SolveParams) * (1 + nl), cudaMemcpyHostToDevice, h->stream));
    if (v1_host)
        for (Part &p : h->parts)
            CUDA_TRY(cudaMemcpyAsync(p.v1buf, v1_host + p.row0, (size_t)p.nrows * 8, cudaMemcpyHostToDevice, h->stream));
    CUDA_TRY(cudaEventRecord(h->ev0, h->stream));
    if (h->use_graph) {
        if (!h->gexec) {
            cudaGraph_t graph;
            int64_t l0 = h->launches;
            CUDA_TRY(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
            h->capturing = true;
            h->prof_next = 0;
            try {
                h->enqueue(h, true);
            } catch (...) {
                h->capturing = false;
                cudaStreamEndCapture(h->stream, &graph);
                throw;
            }
            h->capturing = false;
            CUDA_TRY(cudaStreamEndCapture(h->stream, &graph));
            CUDA_TRY(cudaGraphInstantiate(&h->gexec, graph, 0));
            CUDA_TRY(cudaGraphDestroy(graph));
            h->launches = h->launches - l0;  // kernels per solve
        }
        CUDA_TRY(cudaGraphLaunch(h->gexec, h->stream));
    } else {
        int64_t l0 = h->launches;
        h->prof_next = 0;
        h->enqueue(h, true);
        h->launches = h->launches - l0;
    }
    CUDA_TRY(cudaEventRecord(h->ev1, h->stream));
    for (Part &p : h->parts)
        CUDA_TRY(cudaMemcpyAsync(p.hstate.data(), p.state, p.state_bytes, cudaMemcpyDeviceToHost, h->stream));
}

static void fill_info(topk_eig_s *h, topk_eig_info_t *info) {
    if (!info) return;
    const Part &p = h->parts[0];
    std::memset(info, 0, sizeof(*info));
    const int m_cycle = hget<int>(p, p.st.m_found);  // steps of the last cycle (basis columns used)
    info->iterations = m_cycle;
    info->beta_next = hptr(p, p.st.beta)[m_cycle];   // beta has m + 2 entries; m_cycle <= m
    info->k_found = hget<int>(p, p.st.k_found);
    const int done = hget<int>(p, p.st.done);
    const int nrst = hget<int>(p, p.st.restarts);
    info->restarts = nrst;
    if (nrst > 0)  // total Lanczos steps over the thick-restart cycles (reading Q26)
        info->iterations = h->m + (nrst - 1) * (h->m - h->keep) + (info->iterations - h->keep);
    info->breakdown = done == 1;
    info->converged_stop = done == 2;
    info->conv_checks = h->conv_checks;
    info->reorth_passes = (h->reorth == 3) ? hget<int>(p, p.pro_count) : 0;
    info->jacobi_sweeps = hget<int>(p, p.st.jac_sweeps);
    info->jacobi_converged = hget<int>(p, p.st.jac_conv);
    info->num_parts = h->G;
    float ms = 0.f, ml = 0.f, mj = 0.f, mr = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    cudaEventElapsedTime(&ml, h->ev0, h->evL);
    cudaEventElapsedTime(&mj, h->evL, h->evJ);
    cudaEventElapsedTime(&mr, h->evJ, h->ev1);
    info->ms_solve = ms;
    info->ms_lanczos = ml;
    info->ms_jacobi = mj;
    info->ms_ritz = mr;
    info->bytes_nvlink = h->bytes_nvlink;
    info->bytes_model = h->bytes_model;
    info->gpu_launches = h->launches;
}

#define GUARD(h)                                                                   \
    if (!(h)) return fail(TOPK_E_INVALID, "NULL handle");                          \
    if ((h)->sticky) return fail(TOPK_E_STATE, "handle is in a failed state");    \
    if (cudaSetDevice((h)->device) != cudaSuccess) return fail(TOPK_E_CUDA, "cudaSetDevice failed");

#define CATCH(h)                                                                   \
    catch (CudaFail & e) { (h)->sticky = true; return fail(TOPK_E_CUDA, e.msg); }  \
    catch (NcclFail & e) { (h)->sticky = true; return fail(TOPK_E_NCCL, e.msg); }  \
    catch (std::bad_alloc &) { return fail(TOPK_E_NOMEM, "host allocation failed"); }

extern "C" {

topk_status_t topk_eig_create(topk_eig_t *out, const topk_matrix_t *A, int32_t K, topk_dtype_t storage,
                              topk_dtype_t compute, const topk_eig_opts_t *opts) {
    try {
        return create_impl(out, A, K, storage, compute, opts);
    } catch (std::bad_alloc &) {
        return fail(TOPK_E_NOMEM, "host allocation failed");
    } catch (...) {
        return fail(TOPK_E_INVALID, "unexpected exception in create");
    }
}

topk_status_t topk_eig_solve(topk_eig_t h, uint64_t seed, const double *v1, double *eigenvalues, void *eigenvectors,
                             topk_dtype_t vec_dtype, double *residual_est, topk_eig_info_t *info) {
    GUARD(h);
    if (!eigenvalues) return fail(TOPK_E_INVALID, "eigenvalues must be non-NULL");
    if (eigenvectors && vec_dtype != TOPK_F64 && vec_dtype != TOPK_F32) return fail(TOPK_E_INVALID, "vec_dtype must be F64 or F32");
    try {
        std::vector<void *> outs;
        for (Part &p : h->parts) outs.push_back(eigenvectors ? p.out : nullptr);
        enqueue(h, seed, v1, outs.data(), vec_dtype == TOPK_F32 ? 1 : 0);
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        const Part &p0 = h->parts[0];
        const int kf = hget<int>(p0, p0.st.k_found);
        std::memcpy(eigenvalues, hptr(p0, p0.st.evals), (size_t)h->K * 8);
        if (residual_est) std::memcpy(residual_est, hptr(p0, p0.st.resid), (size_t)h->K * 8);
        if (eigenvectors && h->parts.size() == 1 && h->parts[0].nrows == h->n && kf > 0) {
            // one part holding every row: the K x n block is contiguous on both sides
            const size_t es = vec_dtype == TOPK_F32 ? 4 : 8;
            char *dst = static_cast<char *>(eigenvectors);
            CUDA_TRY(staged_d2h(h->parts[0].out, (size_t)kf * h->n * es,
                                [&](const char *src, size_t off, size_t nb) { par_memcpy(dst + off, src, nb); },
                                h->stream));
        } else if (eigenvectors) {
            const size_t es = vec_dtype == TOPK_F32 ? 4 : 8;
            for (Part &p : h->parts) {
                if (p.nrows == 0 || kf == 0) continue;
                CUDA_TRY(cudaMemcpy2DAsync((char *)eigenvectors + (size_t)p.row0 * es, (size_t)h->n * es, p.out,
                                           (size_t)p.nrows * es, (size_t)p.nrows * es, (size_t)kf, cudaMemcpyDeviceToHost,
                                           h->stream));
            }
            CUDA_TRY(cudaStreamSynchronize(h->stream));
        }
        fill_info(h, info);
    }
    CATCH(h)
    return TOPK_OK;
}

topk_status_t topk_eig_solve_async(topk_eig_t h, uint64_t seed, double *eigenvalues_dev, void *eigenvectors_dev,
                                   topk_dtype_t vec_dtype) {
    GUARD(h);
    if (h->parts.size() != 1 && eigenvectors_dev)
        return fail(TOPK_E_INVALID, "solve_async with eigenvectors needs one local part (G = 1 or multi-process)");
    try {
        void *outs[1] = {eigenvectors_dev};
        std::vector<void *> o(h->parts.size(), nullptr);
        if (eigenvectors_dev) o[0] = outs[0];
        enqueue(h, seed, nullptr, o.data(), vec_dtype == TOPK_F32 ? 1 : 0);
        if (eigenvalues_dev)
            CUDA_TRY(cudaMemcpyAsync(eigenvalues_dev, h->parts[0].st.evals, (size_t)h->K * 8, cudaMemcpyDeviceToDevice, h->stream));
    }
    CATCH(h)
    return TOPK_OK;
}

topk_status_t topk_eig_sync(topk_eig_t h, topk_eig_info_t *info) {
    GUARD(h);
    try {
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        fill_info(h, info);
    }
    CATCH(h)
    return TOPK_OK;
}

topk_status_t topk_eig_kernel_times(topk_eig_t h, double *ms, int32_t *launches) {
    GUARD(h);
    if (!ms || !launches) return fail(TOPK_E_INVALID, "NULL argument");
    if (!h->profile) return fail(TOPK_E_STATE, "create the handle with opts.profile = 1");
    for (int c = 0; c < 8; ++c) { ms[c] = 0.0; launches[c] = 0; }
    try {
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        for (size_t i = 0; i < h->prof_next && i < h->prof.size(); ++i) {
            float t = 0.f;
            CUDA_TRY(cudaEventElapsedTime(&t, h->prof[i].a, h->prof[i].b));
            ms[h->prof[i].cls] += t;
            launches[h->prof[i].cls] += 1;
        }
    }
    CATCH(h)
    return TOPK_OK;
}

void *topk_eig_stream(topk_eig_t h) { return h ? (void *)h->stream : nullptr; }

void topk_eig_destroy(topk_eig_t h) { free_handle(h); }

const char *topk_eig_last_error(void) { return g_last_error.c_str(); }

topk_status_t topk_eig_nccl_id(void *out128) {
    if (!out128) return fail(TOPK_E_INVALID, "NULL out");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(TOPK_E_NCCL, ncclGetErrorString(r));
    std::memcpy(out128, &id, sizeof(id));
    return TOPK_OK;
}

topk_status_t topk_eig_plan_partition(const int64_t *row_ptr, int64_t n, int32_t G, int64_t *boundaries) {
    if (!row_ptr || !boundaries || n < 1) return fail(TOPK_E_INVALID, "bad arguments");
    for (int64_t r = 0; r < n; ++r)
        if (row_ptr[r + 1] < row_ptr[r]) return fail(TOPK_E_STRUCTURE, "row_ptr not monotone");
    topk_status_t s = partition_rule_p(row_ptr, n, G, boundaries);
    if (s != TOPK_OK) return fail(s, "G must be in [1, n]");
    return TOPK_OK;
}

topk_status_t topk_eig_plan_layout(const topk_matrix_t *A, int32_t G, int32_t g, topk_dtype_t storage,
                                   topk_dtype_t values_storage, int64_t *sizes, int64_t *rowptr, int32_t *col,
                                   double *val, int32_t *perm, int32_t *pcol, double *pval, int64_t *chunks,
                                   int64_t *sell, int32_t *items) {
    if (!A) return fail(TOPK_E_INVALID, "A must be non-NULL");
    if (G < 1 || G > 64 || g < 0 || g >= G) return fail(TOPK_E_INVALID, "need 1 <= G <= 64 and 0 <= g < G");
    if (values_storage < TOPK_F64 || values_storage > TOPK_BF16 || storage < TOPK_F64 || storage > TOPK_BF16)
        return fail(TOPK_E_INVALID, "bad dtype");
    try {
        Csr csr;
        std::string err;
        StageClock clk;
        topk_status_t s = canonicalize(*A, csr, err);
        if (s != TOPK_OK) return fail(s, err);
        clk.mark("canonicalize");
        if (G > csr.n) return fail(TOPK_E_INVALID, "G must be <= n");
        std::vector<int64_t> b((size_t)G + 1);
        s = partition_rule_p(csr.rowptr.data(), csr.n, G, b.data());
        if (s != TOPK_OK) return fail(s, "partition failed");
        const int64_t npad = padded_rows(b.data(), G);
        hvec<int32_t> pos;
        degree_order(csr, b.data(), G, pos);
        const hvec<int32_t> colmap = column_map(csr.n, b.data(), G, npad, pos.data());
        clk.mark("partition + order");
        PartLayout L;
        s = build_part(csr, b.data(), G, g, npad, pos.data(), colmap.data(), L, err);
        if (s != TOPK_OK) return fail(s, err);
        clk.mark("build_part");
        auto rv = [&](double x) {
            return values_storage == TOPK_F64 ? x
                   : values_storage == TOPK_F32 ? (double)round_f32(x) : bf16_bits_to_double(round_bf16_bits(x));
        };
        hvec<int32_t> lcol;
        hvec<double> lval;
        logical_from_physical(L, lcol, lval);
        if (sizes) {
            sizes[0] = npad; sizes[1] = L.nrows; sizes[2] = (int64_t)lcol.size(); sizes[3] = L.nnonempty;
            sizes[4] = L.nbig; sizes[5] = (int64_t)L.chunks.size(); sizes[6] = (int64_t)L.sell.size() / 2;
            sizes[7] = (int64_t)L.items.size() / 2; sizes[8] = (int64_t)L.pcol.size();
        }
        if (rowptr)
            for (size_t i = 0; i < L.rowptr.size(); ++i) rowptr[i] = L.rowptr[i];
        if (col) std::memcpy(col, lcol.data(), lcol.size() * 4);
        if (val)
            for (size_t k = 0; k < lval.size(); ++k) val[k] = rv(lval[k]);
        if (perm) std::memcpy(perm, L.perm.data(), L.perm.size() * 4);
        if (pcol) std::memcpy(pcol, L.pcol.data(), L.pcol.size() * 4);
        if (pval)
            for (size_t k = 0; k < L.pval.size(); ++k) pval[k] = rv(L.pval[k]);
        if (chunks)
            for (size_t c = 0; c < L.chunks.size(); ++c) {
                chunks[4 * c] = L.chunks[c].row;
                chunks[4 * c + 1] = L.chunks[c].z0;
                chunks[4 * c + 2] = L.chunks[c].cnt;
                chunks[4 * c + 3] = L.chunks[c].long_id;
            }
        if (sell) std::memcpy(sell, L.sell.data(), L.sell.size() * 8);
        if (items) std::memcpy(items, L.items.data(), L.items.size() * 4);
    } catch (std::bad_alloc &) {
        return fail(TOPK_E_NOMEM, "host allocation failed");
    }
    return TOPK_OK;
}

topk_status_t topk_eig_plan_symmetry(const topk_matrix_t *A, int64_t r0, int64_t r1, uint64_t *sums) {
    if (!A || !sums) return fail(TOPK_E_INVALID, "A and sums must be non-NULL");
    try {
        Csr csr;
        std::string err;
        topk_status_t s = canonicalize(*A, csr, err);
        if (s != TOPK_OK) return fail(s, err);
        if (r0 < 0 || r1 < r0 || r1 > csr.n) return fail(TOPK_E_INVALID, "need 0 <= r0 <= r1 <= n");
        symmetry_sums(csr, r0, r1, sums);
    } catch (std::bad_alloc &) {
        return fail(TOPK_E_NOMEM, "host allocation failed");
    }
    return TOPK_OK;
}

topk_status_t topk_eig_plan_halo(const topk_matrix_t *A, int32_t G, int32_t g, int64_t *n_halo, int64_t *off,
                                 int32_t *pos) {
    if (!A || !n_halo) return fail(TOPK_E_INVALID, "A and n_halo must be non-NULL");
    if (G < 1 || G > 64 || g < 0 || g >= G) return fail(TOPK_E_INVALID, "need 1 <= G <= 64 and 0 <= g < G");
    try {
        Csr csr;
        std::string err;
        topk_status_t s = canonicalize(*A, csr, err);
        if (s != TOPK_OK) return fail(s, err);
        if (G > csr.n) return fail(TOPK_E_INVALID, "G must be <= n");
        std::vector<int64_t> b((size_t)G + 1);
        s = partition_rule_p(csr.rowptr.data(), csr.n, G, b.data());
        if (s != TOPK_OK) return fail(s, "partition failed");
        const int64_t npad = padded_rows(b.data(), G);
        hvec<int32_t> pp;
        degree_order(csr, b.data(), G, pp);
        Halo H;
        build_halo(csr, b.data(), G, g, npad, pp.data(), H);
        *n_halo = H.n;
        if (off) std::memcpy(off, H.off.data(), H.off.size() * 8);
        if (pos && H.n) std::memcpy(pos, H.pos.data(), (size_t)H.n * 4);
    } catch (std::bad_alloc &) {
        return fail(TOPK_E_NOMEM, "host allocation failed");
    }
    return TOPK_OK;
}

topk_status_t topk_eig_export_partition(topk_eig_t h, int64_t *boundaries) {
    if (!h || !boundaries) return fail(TOPK_E_INVALID, "NULL argument");
    std::memcpy(boundaries, h->bounds.data(), h->bounds.size() * 8);
    return TOPK_OK;
}

// one pass's physical arrays back on the host (device column entries, values as double)
static void download_pass(topk_eig_s *h, const SpmvDev &d, std::vector<int32_t> &c, std::vector<double> &v) {
    const size_t zp = (size_t)d.nphys;
    c.assign(zp, 0);
    v.assign(zp, 0.0);
    if (!zp) return;
    CUDA_TRY(scopy(h->stream, c.data(), d.col, zp * 4, cudaMemcpyDeviceToHost));
    if (h->ms == TOPK_F64) {
        CUDA_TRY(scopy(h->stream, v.data(), d.val, zp * 8, cudaMemcpyDeviceToHost));
    } else if (h->ms == TOPK_F32) {
        std::vector<float> f(zp);
        CUDA_TRY(scopy(h->stream, f.data(), d.val, zp * 4, cudaMemcpyDeviceToHost));
        for (size_t k = 0; k < zp; ++k) v[k] = f[k];
    } else {
        std::vector<uint16_t> f(zp);
        CUDA_TRY(scopy(h->stream, f.data(), d.val, zp * 2, cudaMemcpyDeviceToHost));
        for (size_t k = 0; k < zp; ++k) v[k] = bf16_bits_to_double(f[k]);
    }
}

topk_status_t topk_eig_export_layout(topk_eig_t h, int32_t part, int64_t *rowptr, int32_t *col, double *val,
                                     int64_t *n_pad, int64_t *n_rows, int64_t *nnz) {
    GUARD(h);
    if (part < 0 || part >= (int)h->parts.size()) return fail(TOPK_E_INVALID, "bad part");
    Part &p = h->parts[(size_t)part];
    if (n_pad) *n_pad = p.npad;
    if (n_rows) *n_rows = p.nrows;
    if (nnz) *nnz = p.nnz;
    try {
        if (rowptr)
            for (size_t i = 0; i < p.h_rowptr.size(); ++i) rowptr[i] = p.h_rowptr[i];
        if (!col && !val) return TOPK_OK;
        const bool split = p.ypart != nullptr;
        std::vector<int32_t> mc, oc;
        std::vector<double> mv, ov;
        download_pass(h, p.sp, mc, mv);
        std::vector<int32_t> odeg((size_t)std::max<int64_t>(p.nrows, 1), 0);
        if (split) {
            download_pass(h, p.own, oc, ov);
            if (p.nnonempty) CUDA_TRY(scopy(h->stream, odeg.data(), p.owndeg, (size_t)p.nnonempty * 4, cudaMemcpyDeviceToHost));
        }
        std::vector<int32_t> hq;
        if (h->halo) {  // compact entries back to the logical q * n_pad + position (reading Q27)
            hq.resize((size_t)p.nhalo);
            for (int q2 = 0; q2 < h->G; ++q2)
                for (int64_t t2 = p.halo_off[(size_t)q2]; t2 < p.halo_off[(size_t)q2 + 1]; ++t2) hq[(size_t)t2] = q2;
        }
        auto logical_col = [&](int32_t c) -> int32_t {
            if (!h->halo) return c;
            if (c < p.npad) return (int32_t)(p.g * p.npad + c);
            const int64_t e = c - p.npad;
            return (int32_t)(hq[(size_t)e] * p.npad + p.halo_pos_h[(size_t)e]);
        };
        auto slot_of = [&](const SpmvDev &d, int64_t q, int64_t e) -> size_t {
            if (q < p.nbig) return (size_t)(d.h_bigptr[(size_t)q] + e);
            const int64_t sl = (q - p.nbig) / 32, i = (q - p.nbig) % 32;
            return (size_t)(d.h_sell[(size_t)(2 * sl)] + 32 * e + i);
        };
        // a row's entries are in canonical (ascending original column) order; with the
        // split, original columns owned by parts q < g precede the own part's, which precede
        // q > g, so the row is [final-pass entries with owner < g | own-slot pass | the rest]
        for (int64_t q = 0; q < p.nrows; ++q) {
            const int64_t rb = p.h_rowptr[(size_t)q], d = p.h_rowptr[(size_t)q + 1] - rb;
            const int64_t no = split ? odeg[(size_t)q] : 0, nm = d - no;
            int64_t im = 0, k = rb;
            auto put = [&](int32_t c, double v) {
                if (col) col[k] = c;
                if (val) val[k] = v;
                ++k;
            };
            while (split && im < nm && mc[slot_of(p.sp, q, im)] / p.npad < p.g) {
                const size_t sidx = slot_of(p.sp, q, im++);
                put(mc[sidx], mv[sidx]);
            }
            for (int64_t io = 0; io < no; ++io) {
                const size_t sidx = slot_of(p.own, q, io);
                put(oc[sidx], ov[sidx]);
            }
            while (im < nm) {
                const size_t sidx = slot_of(p.sp, q, im++);
                put(logical_col(mc[sidx]), mv[sidx]);
            }
        }
    }
    CATCH(h)
    return TOPK_OK;
}

topk_status_t topk_eig_export_tridiag(topk_eig_t h, double *alpha, double *beta, double *theta_all,
                                      int32_t *m_found) {
    GUARD(h);
    const Part &p = h->parts[0];
    const int mm = hget<int>(p, p.st.m_found);
    if (m_found) *m_found = mm;
    if (alpha) std::memcpy(alpha, hptr(p, p.st.alpha), (size_t)mm * 8);
    if (beta) std::memcpy(beta, hptr(p, p.st.beta), (size_t)(mm + 1) * 8);
    if (theta_all) std::memcpy(theta_all, hptr(p, p.st.theta_all), (size_t)mm * 8);
    return TOPK_OK;
}

static double to_double_elem(const char *base, size_t idx, topk_dtype_t t) {
    if (t == TOPK_F64) return reinterpret_cast<const double *>(base)[idx];
    if (t == TOPK_F32) return reinterpret_cast<const float *>(base)[idx];
    return bf16_bits_to_double(reinterpret_cast<const uint16_t *>(base)[idx]);
}

static topk_status_t export_basis_impl(topk_eig_t h, int32_t part, double *V, int32_t *ncols, bool scaled) {
    GUARD(h);
    if (part < 0 || part >= (int)h->parts.size()) return fail(TOPK_E_INVALID, "bad part");
    Part &p = h->parts[(size_t)part];
    const int mm = hget<int>(p, p.st.m_found);
    const int brk = hget<int>(p, p.st.done);
    const int nc = brk ? mm : mm + 1;
    if (ncols) *ncols = nc;
    if (!V) return TOPK_OK;
    try {
        const size_t es = dsize(h->vs);
        std::vector<char> t((size_t)nc * p.npad * es);
        CUDA_TRY(scopy(h->stream, t.data(), p.V, t.size(), cudaMemcpyDeviceToHost));
        const double *sc = hptr(p, p.st.scale);
        const double *bt = hptr(p, p.st.beta);
        for (int j = 0; j < nc; ++j) {
            const double s = !scaled ? 1.0 : (j < mm) ? sc[j] : 1.0 / bt[mm];
            for (int64_t r = 0; r < p.nrows; ++r)
                V[(size_t)j * p.nrows + p.h_perm[(size_t)r]] = s * to_double_elem(t.data(), (size_t)j * p.npad + r, h->vs);
        }
    }
    CATCH(h)
    return TOPK_OK;
}

topk_status_t topk_eig_export_basis(topk_eig_t h, int32_t part, double *V, int32_t *ncols) {
    return export_basis_impl(h, part, V, ncols, true);
}

topk_status_t topk_eig_export_basis_raw(topk_eig_t h, int32_t part, double *U, int32_t *ncols) {
    return export_basis_impl(h, part, U, ncols, false);
}

topk_status_t topk_eig_debug_spmv(topk_eig_t h, const double *x, double *y) {
    GUARD(h);
    if (!x || !y) return fail(TOPK_E_INVALID, "NULL argument");
    try {
        const size_t es = dsize(h->vs);
        // x rounded to the storage dtype into V column 0 (and the replica)
        std::vector<double> norm((size_t)h->G, 0.0);
        norm[0] = 1.0;  // sum of partials = 1 -> s_1 = 1
        CUDA_TRY(cudaMemcpyAsync(h->ex.norm_part, norm.data(), norm.size() * 8, cudaMemcpyHostToDevice, h->stream));
        for (Part &p : h->parts) {
            std::vector<char> buf((size_t)p.npad * es, 0);
            for (int64_t r = 0; r < p.nrows; ++r) {
                const double v = x[p.row0 + p.h_perm[(size_t)r]];
                if (h->vs == TOPK_F64) reinterpret_cast<double *>(buf.data())[r] = v;
                else if (h->vs == TOPK_F32) reinterpret_cast<float *>(buf.data())[r] = round_f32(v);
                else reinterpret_cast<uint16_t *>(buf.data())[r] = round_bf16_bits(v);
            }
            CUDA_TRY(scopy(h->stream, p.V, buf.data(), buf.size(), cudaMemcpyHostToDevice));
            if (h->G > 1 && h->comm == nullptr)
                CUDA_TRY(scopy(h->stream, rep_slot(h, p), buf.data(), buf.size(), cudaMemcpyHostToDevice));
            if (h->comm) CUDA_TRY(scopy(h->stream, rep_slot(h, p), buf.data(), buf.size(), cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemsetAsync(p.st.done, 0, sizeof(int), h->stream));
            CUDA_TRY(cudaMemsetAsync(p.st.tscale, 0, sizeof(double), h->stream));
            if (!p.y_dbg) p.y_dbg = h->alloc<double>((size_t)std::max<int64_t>(p.nrows, 1));
        }
        if (h->comm || h->halo) exch_vec_norm(h);
        for (Part &p : h->parts) h->spmv_only(h, p);
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        for (Part &p : h->parts) {
            std::vector<double> t((size_t)p.nrows);
            CUDA_TRY(scopy(h->stream, t.data(), p.y_dbg, (size_t)p.nrows * 8, cudaMemcpyDeviceToHost));
            for (int64_t r = 0; r < p.nrows; ++r) y[p.row0 + p.h_perm[(size_t)r]] = t[(size_t)r];
        }
    }
    CATCH(h)
    return TOPK_OK;
}

size_t topk_eig_trim_pool(void) { return topk::pool_trim(); }

}  // extern "C"
