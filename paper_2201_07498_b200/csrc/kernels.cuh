// kernels.cuh — the hot path of arXiv 2201.07498 as sm_100a kernels.
//
// Per Lanczos iteration i (Algorithm 1) on each part g:
//   k_spmv     Alg.1 l.6-7 (beta_i from the previous norm partials, deferred
//              normalisation) + l.9 SpMV y = M_g v_i + l.10 alpha partial
//   k_step     l.10 alpha sum over parts + l.11 three-term recurrence
//              w = y - alpha_i v_i - beta_i v_{i-1} + l.12-18 reorth dots
//              h_j = v_j . w (skinny multi-dot over the stored basis)
//   k_correct  l.15/18 correction u_{i+1} = w - sum_j h_j v_j, rounded once
//              to the storage dtype, + its squared norm (next beta, l.6)
// then k_jacobi and k_ritz / k_ritz_norm.
//
// Deferred normalisation: the basis is stored unnormalised (column c holds
// u_{c+1}); v_{c+1} = s_c u_{c+1} with s_c = 1/beta_{c+1} kept in fp64 and
// applied by every consumer. This is Alg.1's order (beta_i and v_i are formed at
// the top of iteration i, l.5-7) with the division folded into the readers.
//
// Reductions are deterministic: fixed-shape shuffle trees, fixed warp order,
// per-block slots summed in block order by the last-arriving block, and
// cross-part sums in rank order (no floating-point atomics).
#pragma once
#include <cooperative_groups.h>

#include "device_common.cuh"
#include "host_prep.h"

namespace topk {

constexpr int kNT = 256;  // threads per block for the streaming kernels
constexpr int kSpmvNT = 256;  // SpMV CTA size (occupancy-limited grid, no shared memory)
#ifndef TOPK_RITZ_KB
#define TOPK_RITZ_KB 8
#endif
constexpr int kRitzKB = TOPK_RITZ_KB;  // Ritz outputs per thread (dev knob, tools/build.py build_variant)
constexpr int kStepJB = 16;  // basis columns per multi-dot pass of k_step (reorth-off path)
#ifndef TOPK_STEP_MAXNC
#define TOPK_STEP_MAXNC 17
#endif
constexpr int kStepMaxNC = TOPK_STEP_MAXNC;  // widest exact-width multi-dot pass (k_stepw; dev build variant)
#ifndef TOPK_CORR_MAXNC
#define TOPK_CORR_MAXNC 17  // 24 measured the same on C3 (tools/lab/spmv_variants.py)
#endif
constexpr int kCorrMaxNC = TOPK_CORR_MAXNC;  // widest exact-width correction (k_correctw)

struct LzState {
    double *alpha;      // [m]     alpha_1..alpha_m
    double *beta;       // [m+2]   beta[0] = beta_1 = 0, beta[k] = beta_{k+1}
    double *scale;      // [m+1]   s_c = 1/beta_{c+1}: v_{c+1} = s_c u_{c+1}
    double *tscale;     // [1]     max(|alpha_1..|, beta_2..) so far (reading Q7)
    int *done;          // [1]     breakdown flag
    int *m_found;       // [1]     completed iterations m'
    int *k_found;       // [1]
    int *jac_sweeps;    // [1]
    int *jac_conv;      // [1]
    double *theta_all;  // [m]
    double *evals;      // [K]
    double *coefS;      // [m*K]   sign-fixed S[j, sel_k] * s_j (Ritz coefficients)
    double *resid;      // [K]
    double *gram;       // [m*m] G_jl = u_j . u_l of the stored (unnormalised) basis, summed over parts
    double *rnrm2;      // [K] ||y_k||^2 of the selected Ritz vectors from the Gram matrix
    int use_gram;       // 1: Ritz norms from the Gram matrix (reading Q24), 0: Ritz pass 0
    int m;
    double tau;
    // thick restart (reading Q26): after a restart T is [[diag(theta), b], [b^T, tridiag]]
    int *arrow_k;       // [1]     0: plain tridiagonal T; k: rows/cols [0, k) are the kept Ritz pairs
    int *restarts;      // [1]     restarts done in this solve
    double *arrow_theta;// [keep]  kept Ritz values (diagonal of T[0:k, 0:k])
    double *arrow_b;    // [keep]  coupling b_j = beta_{m+1} s_{m,j} (T[j][k] = T[k][j])
    double *coefR;      // [m*keep] S[l, J_j] * s_l: kept Ritz vectors in the stored basis
    int keep;           // kept pairs per restart (0: off)
};

struct Exch {            // cross-part exchange buffers, slot g written by part g
    double *alpha_part;  // [G]
    double *hpart;       // [G][2 (m+1)]: reorth dots h_j at [0, m+1), Gram u_j . u_i at [m+1, 2 (m+1))
    double *norm_part;   // [G]
    double *ritz_part;   // [G][K]
    double *rst_part;    // [G][keep] squared norms of the stored restart vectors
    void *replica;       // [G * npad] storage dtype (G > 1)
};

// ---------------------------------------------------------------------------
// Top of iteration `it` (Alg.1 l.5-7): beta_it = ||u_it|| from the G norm
// partials (rank order), breakdown test, s = 1/beta. Returns false if the
// kernel must not run (already done, or breakdown now).
__device__ __forceinline__ bool lz_prologue(int it, const LzState &st, const Exch &ex, int G,
                                            double &s) {
    if (*(volatile int *)st.done) return false;
    double sq = 0.0;
    for (int q = 0; q < G; ++q) sq += __ldcg(ex.norm_part + q);
    const double b = sqrt(sq);
    const bool lead = (blockIdx.x == 0 && threadIdx.x == 0);
    const bool brk = (it == 1) ? !(sq > 0.0) : (b <= st.tau * *st.tscale);
    if (brk) {
        if (lead) {
            *st.done = 1;
            *st.m_found = it - 1;
            st.beta[it - 1] = (it == 1) ? 0.0 : b;
        }
        return false;
    }
    s = 1.0 / b;
    if (lead) {
        st.beta[it - 1] = (it == 1) ? 0.0 : b;
        st.scale[it - 1] = s;
        st.gram[(size_t)(it - 1) * st.m + (it - 1)] = sq;  // ||u_it||^2 (Gram diagonal)
        *st.m_found = it;
    }
    return true;
}

// ---------------------------------------------------------------------------
// a5: start vector (PAPER.md:65,75 "L2-normalized random vector"; :205).
struct V1Args {
    void *u0;              // V column 0 (npad)
    void *rep_slot;        // replica slot g or nullptr
    const uint64_t *seed;  // device param
    const int *use_v1;     // device param
    const double *v1;      // device, n_g doubles in original row order (if *use_v1)
    const int32_t *perm;   // position -> part-local original row (hub-first order)
    int64_t row0, nrows, npad;
    double *slots;
    unsigned *counter;
    LzState st;
    Exch ex;
    int g;
};

template <typename ST, typename CT>
__global__ void __launch_bounds__(kNT) k_v1(V1Args a) {
    __shared__ double red_storage[kNT / 32];  // CT partials, or doubles for the final sums
    CT *red = reinterpret_cast<CT *>(red_storage);
    __shared__ int sflag;
    constexpr int VW = Vw<ST>::N;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.st.done = 0;
        *a.st.m_found = 0;
        *a.st.tscale = 0.0;
        *a.st.arrow_k = 0;
        *a.st.restarts = 0;
    }
    const uint64_t seed = *a.seed;
    const int use_v1 = *a.use_v1;
    const uint64_t hs = mix64(mix64(seed) ^ 0x7631ull);
    CT nrm = CT(0);
    const int64_t nvec = a.npad / VW;
    for (int64_t v = (int64_t)blockIdx.x * kNT + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * kNT) {
        CT u[VW];
#pragma unroll
        for (int q = 0; q < VW; ++q) {
            const int64_t r = v * VW + q;
            double x = 0.0;
            if (r < a.nrows) {
                const int32_t orow = __ldg(a.perm + r);
                if (use_v1) x = a.v1[orow];
                else {
                    uint64_t h = mix64(hs ^ (uint64_t)(a.row0 + orow));
                    x = 2.0 * ((double)(h >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
                }
            }
            u[q] = (CT)x;
        }
        vstore_back<ST, CT>(reinterpret_cast<ST *>(a.u0) + v * VW, u);
        if (a.rep_slot) vstore<ST, CT>(reinterpret_cast<ST *>(a.rep_slot) + v * VW, u);
#pragma unroll
        for (int q = 0; q < VW; ++q) nrm += u[q] * u[q];
    }
    CT t = block_sum<CT, kNT>(nrm, red);
    if (threadIdx.x == 0) a.slots[blockIdx.x] = (double)t;
    if (arrive_last(a.counter, &sflag)) {
        double tot = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, red_storage);
        if (threadIdx.x == 0) {
            a.ex.norm_part[a.g] = tot;
            *a.counter = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// a7: SpMV + alpha partial (Alg.1 l.9-10) on the physical format of
// host_prep.h (rows in degree order):
//  * big rows (degree > kSellMaxLen): warp per chunk of <= kChunkNnz nonzeros,
//    lanes stride the row with coalesced loads, warp shuffle reduction; a row
//    of several chunks is finished by its last-arriving chunk in chunk order;
//  * SELL-32 slices: lane per row, entry e of the slice's 32 rows is one
//    coalesced 128-byte load of col and of val, no reduction at all.
// x gathers are plain L1-cached loads: in degree order the hub columns are the
// dense prefix of x, so they stay L1-resident while col/val are streamed with
// L1::no_allocate (measured on B200 to beat a shared-memory hub cache 2x, see
// DESIGN.md section 7); C3's 16.8 MB x is L2-resident. Products
// and sums in the compute dtype (reading Q14). Epilogue per row: y_r = s_i *
// sum (deferred normalisation), stored once rounded, alpha partial
// y_r * s_i * u_i[r]. Deterministic: fixed orders and shuffle trees.
struct SpmvArgs {
    const int32_t *col;   // physical
    const void *val;      // physical
    const Chunk *chunks;  // [nchunks] (64-bit first nonzero: parts may hold >= 2^31 nonzeros)
    const int4 *longrows; // [nlong] LongRow
    const longlong2 *sell; // [nslices] (base, width)
    const int2 *items;    // [nitems] (first slice, end slice)
    int nchunks, nitems, nbig, nnonempty, nlong;
    double *long_parts;   // [nchunks]
    unsigned *long_cnt;   // [nlong]
    double *alpha_long;   // [nlong]
    const void *x;        // gather source: V column it-1 (G = 1) or the replica
    int64_t xlen;         // elements of x (TOPK_CHECKS bounds)
    double *ypart;        // two-pass SpMV (overlapped exchange): own-slot row sums, written by the
                          // first pass, added by the final one; nullptr: one pass
    const void *ui;       // local u_it (V column it-1)
    void *y;              // v_tmp (Q2), storage dtype
    double *y_dbg;        // optional fp64 unscaled row sums (debug export)
    double *slots;        // [grid]
    unsigned *counter;
    LzState st;
    Exch ex;
    int G, g;
};

template <typename VT> __device__ __forceinline__ VT ld_val_stream(const VT *p);
template <> __device__ __forceinline__ float ld_val_stream<float>(const float *p) { return ld_noalloc<float>(p); }
template <> __device__ __forceinline__ double ld_val_stream<double>(const double *p) { return ld_noalloc<double>(p); }
template <> __device__ __forceinline__ bf16 ld_val_stream<bf16>(const bf16 *p) { return ld_noalloc<bf16>(p); }
__device__ __forceinline__ int ld_col_stream(const int32_t *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

template <typename VT, typename ST, typename CT, bool LOCAL, bool BIG, int GQ>
// GQ: nonzeros per lane per group (the next group's col/val are in flight while the
// current group's x gathers are).
// BIG = false: a pass without big-row chunks (low-degree matrices: meshes, road
// networks); the chunk path is compiled out, which frees registers for more resident
// warps (the host picks the instantiation from the pass's chunk count).
// LOCAL: the first pass of the two-pass SpMV: only the own-slot
// columns, which do not wait for the vector exchange; unscaled fp64 row sums to
// ypart, no alpha, no state writes. Otherwise the final (or only) pass, which adds
// ypart (when set) before the epilogue.
// dev knobs (tools/build.py build_variant): prefetch depth and an optional
// min-blocks bound. Measured on C3 (tools/lab/spmv_variants.py): GQ 8 with the plain
// bound (80 registers, 3 CTAs/SM) 229 us; GQ 4 / 6 at 4 CTAs/SM 229 / 232 us; an
// explicit (256, 1) bound makes ptxas take 94 registers (2 CTAs/SM): 256 us.
#ifndef TOPK_SPMV_GQ
#define TOPK_SPMV_GQ 8
#endif
#ifndef TOPK_SPMV_SELL_PIPE3
#define TOPK_SPMV_SELL_PIPE3 1
#endif
#ifdef TOPK_SPMV_MINB
#define TOPK_SPMV_BOUNDS __launch_bounds__(kSpmvNT, TOPK_SPMV_MINB)
#else
#define TOPK_SPMV_BOUNDS __launch_bounds__(kSpmvNT)
#endif
__device__ __forceinline__ void spmv_body(const SpmvArgs &a, int it) {
    __shared__ CT red[kSpmvNT / 32];
    __shared__ double redd[kSpmvNT / 32];
    __shared__ int sflag;

    double sd = 1.0;
    if constexpr (LOCAL) {
        if (*(volatile int *)a.st.done) return;  // no state writes: the final pass does them
    } else {
        if (!lz_prologue(it, a.st, a.ex, a.G, sd)) return;
    }
    const CT s = (CT)sd;
    const double *__restrict__ yp = a.ypart;
    const int lane = threadIdx.x & 31;
    const int gwarp = (int)((blockIdx.x * kSpmvNT + threadIdx.x) >> 5);
    const int nwarps = (int)(gridDim.x * (kSpmvNT / 32));
    const VT *__restrict__ val = reinterpret_cast<const VT *>(a.val);
    const int32_t *__restrict__ col = a.col;
    const ST *__restrict__ x = reinterpret_cast<const ST *>(a.x);
    const ST *__restrict__ ui = reinterpret_cast<const ST *>(a.ui);
    ST *__restrict__ y = reinterpret_cast<ST *>(a.y);
    CT alpha_acc = CT(0);
    const int nwork = a.nchunks + a.nitems;
    for (int wi = gwarp; wi < nwork; wi += nwarps) {
        if (BIG && wi < a.nchunks) {
            // ---- big-row chunk: lane stream k = zb + lane + 32 t, warp reduction
            const Chunk *Cp = a.chunks + wi;
            const int64_t zb = __ldg(&Cp->z0);
            const int crow = __ldg(&Cp->row), ccnt = __ldg(&Cp->cnt), clid = __ldg(&Cp->long_id);
            const int nt = (ccnt - lane + 31) / 32;  // this lane's element count
            CT acc0 = CT(0), acc1 = CT(0);
            int cc[GQ];
            VT vv[GQ];
#pragma unroll
            for (int q = 0; q < GQ; ++q) {
                const int64_t k = zb + lane + 32 * q;
                cc[q] = q < nt ? ld_col_stream(col + k) : 0;
                vv[q] = q < nt ? ld_val_stream<VT>(val + k) : VT(0);
            }
            for (int t0 = 0; t0 < nt; t0 += GQ) {
                ST xg[GQ];  // raw storage values, converted at use
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    TOPK_DCHECK(t0 + q >= nt || (cc[q] >= 0 && cc[q] < a.xlen), "SpMV chunk gather out of x");
                    xg[q] = (t0 + q < nt) ? __ldg(x + cc[q]) : ST(0);
                }
                VT vc[GQ];
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    vc[q] = vv[q];
                    const int t = t0 + GQ + q;
                    const int64_t k = zb + lane + 32 * t;
                    cc[q] = t < nt ? ld_col_stream(col + k) : 0;
                    vv[q] = t < nt ? ld_val_stream<VT>(val + k) : VT(0);
                }
#pragma unroll
                for (int q = 0; q < GQ; q += 2) {
                    acc0 += cvt<CT>(vc[q]) * cvt<CT>(xg[q]);
                    acc1 += cvt<CT>(vc[q + 1]) * cvt<CT>(xg[q + 1]);
                }
            }
            CT part = warp_sum(acc0 + acc1);
            if (lane == 0) {
                if (clid < 0) {
                    TOPK_DCHECK(crow >= 0 && crow < a.nbig, "big-row position");
                    if constexpr (LOCAL) {
                        a.ypart[crow] = (double)part;
                    } else {
                        if (yp) part += (CT)__ldcg(yp + crow);
                        const CT yv = s * part;
                        y[crow] = rnd_ct<ST, CT>(yv);
                        alpha_acc += yv * (s * cvt<CT>(ui[crow]));
                        if (a.y_dbg) a.y_dbg[crow] = (double)part;
                    }
                } else {
                    const int4 L = __ldg(a.longrows + clid);
                    a.long_parts[wi] = (double)part;
                    __threadfence();
                    const unsigned prev = atomicAdd(a.long_cnt + clid, 1u);
                    TOPK_DCHECK(prev < (unsigned)L.z && crow == L.x, "long-row ticket");
                    if (prev == (unsigned)L.z - 1) {
                        __threadfence();
                        CT sum = CT(0);
                        for (int q = 0; q < L.z; ++q) sum += (CT)__ldcg(a.long_parts + L.y + q);
                        if constexpr (LOCAL) {
                            a.ypart[L.x] = (double)sum;
                        } else {
                            if (yp) sum += (CT)__ldcg(yp + L.x);
                            const CT yv = s * sum;
                            y[L.x] = rnd_ct<ST, CT>(yv);
                            a.alpha_long[clid] = (double)(yv * (s * cvt<CT>(ui[L.x])));
                            if (a.y_dbg) a.y_dbg[L.x] = (double)sum;
                        }
                        a.long_cnt[clid] = 0u;
                    }
                }
            }
        } else {
            // ---- SELL-32 slices of this item: their storage is contiguous, so lane l
            // streams base + 32 t + l for t = 0 .. sum(w) - 1; slice boundaries are
            // warp-uniform (row result emitted, accumulator reset)
            const int2 I = __ldg(a.items + (wi - a.nchunks));
            const int64_t base = __ldg(a.sell + I.x).x;
            const longlong2 Sl = __ldg(a.sell + (I.y - 1));
            const int ntot = (int)((Sl.x - base) / 32 + Sl.y);  // total width of the item
            int sl = I.x;
            int bound = (int)__ldg(a.sell + sl).y;  // t at which slice sl ends
            // one slice ahead: the next slice's width, and this slice's epilogue inputs
            // (u_i and the own-pass partial of its row), so that low-degree slices (a few
            // entries each) do not wait on a dependent load at every slice end
            int wnext = (sl + 1 < I.y) ? (int)__ldg(a.sell + sl + 1).y : 0;
            int row = a.nbig + 32 * sl + lane;
            ST ucur = ST(0);
            double ypc = 0.0;
            if constexpr (!LOCAL) {
                if (row < a.nnonempty) {
                    ucur = ld_noalloc<ST>(ui + row);
                    if (yp) ypc = __ldcg(yp + row);
                }
            }
            CT acc = CT(0);
          if constexpr (!BIG && TOPK_SPMV_SELL_PIPE3) {
            // SELL-only kernel: three-stage software pipeline -- col/val loads two groups
            // ahead, x gathers one group ahead of the multiply-adds, so a gather never
            // waits on a column index loaded in the same step (low-degree slices have
            // little else to overlap; profiles/r02_mesh_spmv_ab.jsonl)
            int cB[GQ], cC[GQ];
            VT vA[GQ], vB[GQ], vC[GQ];
            ST xA[GQ], xB[GQ];
#pragma unroll
            for (int q = 0; q < GQ; ++q) {
                const int64_t k = base + lane + 32 * q;
                const int c0 = q < ntot ? ld_col_stream(col + k) : 0;
                vA[q] = q < ntot ? ld_val_stream<VT>(val + k) : VT(0);
                const int t1 = GQ + q;
                cB[q] = t1 < ntot ? ld_col_stream(col + k + 32 * GQ) : 0;
                vB[q] = t1 < ntot ? ld_val_stream<VT>(val + k + 32 * GQ) : VT(0);
                TOPK_DCHECK(q >= ntot || (c0 >= 0 && c0 < a.xlen), "SpMV SELL gather out of x");
                xA[q] = q < ntot ? __ldg(x + c0) : ST(0);
            }
            for (int t0 = 0; t0 < ntot; t0 += GQ) {
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    const int t1 = t0 + GQ + q, t2 = t0 + 2 * GQ + q;
                    TOPK_DCHECK(t1 >= ntot || (cB[q] >= 0 && cB[q] < a.xlen), "SpMV SELL gather out of x");
                    xB[q] = t1 < ntot ? __ldg(x + cB[q]) : ST(0);
                    const int64_t k = base + lane + 32 * t2;
                    cC[q] = t2 < ntot ? ld_col_stream(col + k) : 0;
                    vC[q] = t2 < ntot ? ld_val_stream<VT>(val + k) : VT(0);
                }
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    const int t = t0 + q;
                    if (t < ntot) {
                        acc += cvt<CT>(vA[q]) * cvt<CT>(xA[q]);
                        if (t + 1 == bound) {  // warp-uniform: slice sl complete
                            if (row < a.nnonempty) {
                                if constexpr (LOCAL) {
                                    a.ypart[row] = (double)acc;
                                } else {
                                    if (yp) acc += (CT)ypc;
                                    const CT yv = s * acc;
                                    y[row] = rnd_ct<ST, CT>(yv);
                                    alpha_acc += yv * (s * cvt<CT>(ucur));
                                    if (a.y_dbg) a.y_dbg[row] = (double)acc;
                                }
                            }
                            acc = CT(0);
                            ++sl;
                            bound += wnext;
                            wnext = (sl + 1 < I.y) ? (int)__ldg(a.sell + sl + 1).y : 0;
                            row += 32;
                            if constexpr (!LOCAL) {
                                if (row < a.nnonempty) {
                                    ucur = ld_noalloc<ST>(ui + row);
                                    if (yp) ypc = __ldcg(yp + row);
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < GQ; ++q) { xA[q] = xB[q]; vA[q] = vB[q]; vB[q] = vC[q]; cB[q] = cC[q]; }
            }
          } else {
            int cc[GQ];
            VT vv[GQ];
#pragma unroll
            for (int q = 0; q < GQ; ++q) {
                const int64_t k = base + lane + 32 * q;
                cc[q] = q < ntot ? ld_col_stream(col + k) : 0;
                vv[q] = q < ntot ? ld_val_stream<VT>(val + k) : VT(0);
            }
            for (int t0 = 0; t0 < ntot; t0 += GQ) {
                ST xg[GQ];  // raw storage values, converted at use
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    TOPK_DCHECK(t0 + q >= ntot || (cc[q] >= 0 && cc[q] < a.xlen), "SpMV SELL gather out of x");
                    xg[q] = (t0 + q < ntot) ? __ldg(x + cc[q]) : ST(0);
                }
                VT vc[GQ];
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    vc[q] = vv[q];
                    const int t = t0 + GQ + q;
                    const int64_t k = base + lane + 32 * t;
                    cc[q] = t < ntot ? ld_col_stream(col + k) : 0;
                    vv[q] = t < ntot ? ld_val_stream<VT>(val + k) : VT(0);
                }
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    const int t = t0 + q;
                    if (t < ntot) {
                        acc += cvt<CT>(vc[q]) * cvt<CT>(xg[q]);
                        if (t + 1 == bound) {  // warp-uniform: slice sl complete
                            if (row < a.nnonempty) {
                                if constexpr (LOCAL) {
                                    a.ypart[row] = (double)acc;
                                } else {
                                    if (yp) acc += (CT)ypc;
                                    const CT yv = s * acc;
                                    y[row] = rnd_ct<ST, CT>(yv);
                                    alpha_acc += yv * (s * cvt<CT>(ucur));
                                    if (a.y_dbg) a.y_dbg[row] = (double)acc;
                                }
                            }
                            acc = CT(0);
                            ++sl;
                            bound += wnext;
                            wnext = (sl + 1 < I.y) ? (int)__ldg(a.sell + sl + 1).y : 0;
                            row += 32;
                            if constexpr (!LOCAL) {
                                if (row < a.nnonempty) {
                                    ucur = ld_noalloc<ST>(ui + row);
                                    if (yp) ypc = __ldcg(yp + row);
                                }
                            }
                        }
                    }
                }
            }
          }
        }
    }
    if constexpr (LOCAL) return;
    const CT tot = block_sum<CT, kSpmvNT>(alpha_acc, red);
    if (threadIdx.x == 0) a.slots[blockIdx.x] = (double)tot;
    if (arrive_last(a.counter, &sflag)) {
        const double s1 = block_sum_array<double, kSpmvNT>(a.slots, gridDim.x, 1, redd);
        const double s2 = block_sum_array<double, kSpmvNT>(a.alpha_long, a.nlong, 1, redd);
        if (threadIdx.x == 0) {
            a.ex.alpha_part[a.g] = s1 + s2;
            *a.counter = 0u;
        }
    }
}

// The SpMV kernels: with the big-row chunk path (plain bound; measured above), and
// SELL-only (a pass without chunks: low-degree matrices such as meshes and road
// networks). Measured on C6 (tools/lab/spmv_ab.py, profiles/r02_mesh_spmv_ab.jsonl),
// two-stage loop: (min CTAs/SM, GQ) = (3, 8) 167-171 us, (4, 4) 172, (3, 6) 176,
// (6, 2) 186, (5, 4) 198, (2, 16) 199, (4, 2) 226, (6, 4) 257 (spills); the stream marked
// L2 evict-first: 194 vs 172 (worse). Three-stage loop (adopted): (4, 4) 161.6-161.7 us,
// (3, 8) 164.5, (3, 6) 170, (5, 3) 183 and (6, 2) 211 (spills).
#ifndef TOPK_SPMV_SELL_MINB
#define TOPK_SPMV_SELL_MINB 4
#endif
#ifndef TOPK_SPMV_SELL_GQ
#define TOPK_SPMV_SELL_GQ 4
#endif
template <typename VT, typename ST, typename CT, bool LOCAL>
__global__ void TOPK_SPMV_BOUNDS k_spmv(SpmvArgs a, int it) {
    spmv_body<VT, ST, CT, LOCAL, true, TOPK_SPMV_GQ>(a, it);
}
template <typename VT, typename ST, typename CT, bool LOCAL>
__global__ void __launch_bounds__(kSpmvNT, (sizeof(VT) == 8 || sizeof(ST) == 8) ? 3 : TOPK_SPMV_SELL_MINB)
    k_spmv_sell(SpmvArgs a, int it) {  // fp64 storage: 3 CTAs/SM (the 4-CTA bound spills)
    spmv_body<VT, ST, CT, LOCAL, false, TOPK_SPMV_SELL_GQ>(a, it);
}

// ---------------------------------------------------------------------------
// a9: fused step (Alg.1 l.10 sum, l.11, l.12-18 dots). mode 0: recurrence +
// multi-dot (reorth on); mode 1: recurrence only, w published as u_{i+1} with its
// norm (reorth off, PAPER.md:123 optional); mode 2: multi-dot of the freshly
// corrected column `it` (second CGS pass).
struct StepArgs {
    const void *y;      // v_tmp
    void *w;            // v_nxt (mode 0) / unused
    const void *V;      // basis, column stride npad
    void *vout;         // mode 1: V column it; mode 2: unused
    void *rep_slot;     // mode 1 publish (G > 1)
    int64_t npad;
    int ld;             // m + 1 (slot stride)
    double *slots;      // [grid][ld]
    unsigned *counter;
    LzState st;
    Exch ex;
    int G, g, mode;
    int no_prev;        // first step after a thick restart: no beta_i v_{i-1} term (reading Q26)
    const int *gate;    // partial reorthogonalisation (reading Q29): run only if *gate != 0
};

template <typename ST, typename CT, int JB>
__global__ void __launch_bounds__(kNT, 2) k_step(StepArgs a, int it) {
    constexpr int VW = Vw<ST>::N;
    __shared__ CT part[kNT / 32][JB];
    __shared__ double red_storage[kNT / 32];  // CT partials, or doubles for the final sums
    CT *red = reinterpret_cast<CT *>(red_storage);
    __shared__ int sflag;
    if (*(volatile int *)a.st.done) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const ST *__restrict__ V = reinterpret_cast<const ST *>(a.V);
    const int64_t nvec = a.npad / VW;
    CT c1 = CT(0), c2 = CT(0);
    if (a.mode != 2) {
        double al = 0.0;
        for (int q = 0; q < a.G; ++q) al += __ldcg(a.ex.alpha_part + q);  // l.10, rank order
        const double bi = a.st.beta[it - 1];
        if (blockIdx.x == 0 && tid == 0) {
            a.st.alpha[it - 1] = al;
            double ts = *a.st.tscale;
            ts = fmax(ts, fabs(al));
            ts = fmax(ts, bi);
            *a.st.tscale = ts;
        }
        c1 = (CT)(al * a.st.scale[it - 1]);                       // alpha_i * s_i
        c2 = (it > 1 && !a.no_prev) ? (CT)(bi * a.st.scale[it - 2]) : CT(0);    // beta_i * s_{i-1}
    }
    const ST *ucur = V + (size_t)(it - 1) * a.npad;
    const ST *uprev = V + (size_t)(it > 1 ? it - 2 : 0) * a.npad;
    const ST *yv = reinterpret_cast<const ST *>(a.y);
    ST *wv = reinterpret_cast<ST *>(a.w);
    const ST *src2 = V + (size_t)it * a.npad;  // mode 2 input column

    if (a.mode == 1) {  // no reorth: w -> u_{i+1}, norm partial
        CT nrm = CT(0);
        ST *out = reinterpret_cast<ST *>(a.vout);
        for (int64_t v = (int64_t)blockIdx.x * kNT + tid; v < nvec; v += (int64_t)gridDim.x * kNT) {
            CT yy[VW], u1[VW], u0[VW], w[VW];
            vload<ST, CT>(yv + v * VW, yy);
            vload<ST, CT>(ucur + v * VW, u1);
            if (it > 1) vload<ST, CT>(uprev + v * VW, u0);
#pragma unroll
            for (int q = 0; q < VW; ++q) w[q] = yy[q] - c1 * u1[q] - (it > 1 ? c2 * u0[q] : CT(0));
            vstore_back<ST, CT>(out + v * VW, w);
            if (a.rep_slot) vstore<ST, CT>(reinterpret_cast<ST *>(a.rep_slot) + v * VW, w);
#pragma unroll
            for (int q = 0; q < VW; ++q) nrm += w[q] * w[q];
        }
        const CT tb = block_sum<CT, kNT>(nrm, red);
        if (tid == 0) a.slots[blockIdx.x] = (double)tb;
        if (arrive_last(a.counter, &sflag)) {
            const double tot = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, red_storage);
            if (tid == 0) { a.ex.norm_part[a.g] = tot; *a.counter = 0u; }
        }
        return;
    }

    // Multi-dot h_j = u_j . w in passes over blocks of JB basis columns: a thread
    // issues the loads of all JB columns of its row-vector at once (memory-level
    // parallelism; measured ~6.2 TB/s for a 16-column block on B200), the first
    // pass also forms w (recurrence) and stores it, later passes re-read w (L2).
    // balanced passes: it columns in ceil(it / JB) passes of equal width
    const int npass = (it + JB - 1) / JB, width = (it + npass - 1) / npass;
    for (int j0 = 0; j0 < it; j0 += width) {
        const int jend = min(it, j0 + width);
        CT acc[JB];
#pragma unroll
        for (int q = 0; q < JB; ++q) acc[q] = CT(0);
        for (int64_t v = (int64_t)blockIdx.x * kNT + tid; v < nvec; v += (int64_t)gridDim.x * kNT) {
            uint4 u[JB];  // raw 16-byte storage vectors, converted at use (register budget)
#pragma unroll
            for (int q = 0; q < JB; ++q)
                if (j0 + q < jend) u[q] = __ldg(reinterpret_cast<const uint4 *>(V + (size_t)(j0 + q) * a.npad + v * VW));
            CT w[VW];
            if (a.mode == 2) {
                vload<ST, CT>(src2 + v * VW, w);
            } else if (j0 == 0) {
                CT yy[VW], u1[VW], u0[VW];
                vload<ST, CT>(yv + v * VW, yy);
                vload<ST, CT>(ucur + v * VW, u1);
                if (it > 1) vload<ST, CT>(uprev + v * VW, u0);
#pragma unroll
                for (int q = 0; q < VW; ++q) w[q] = yy[q] - c1 * u1[q] - (it > 1 ? c2 * u0[q] : CT(0));
                vstore_back<ST, CT>(wv + v * VW, w);  // w rounded once; dots use what was stored
            } else {
                vload<ST, CT>(wv + v * VW, w);
            }
#pragma unroll
            for (int q = 0; q < JB; ++q) {
                if (j0 + q < jend) {
                    const ST *ue = reinterpret_cast<const ST *>(&u[q]);
                    CT d = CT(0);
#pragma unroll
                    for (int e = 0; e < VW; ++e) d += cvt<CT>(ue[e]) * w[e];
                    acc[q] += d;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < JB; ++q) {
            const CT r = warp_sum(acc[q]);
            if (lane == 0) part[wid][q] = r;
        }
        __syncthreads();
        if (tid < JB && j0 + tid < jend) {
            CT r = CT(0);
#pragma unroll
            for (int w8 = 0; w8 < kNT / 32; ++w8) r += part[w8][tid];
            a.slots[(size_t)blockIdx.x * a.ld + j0 + tid] = (double)r;
        }
        __syncthreads();
    }
    if (arrive_last(a.counter, &sflag)) {
        // warp w sums column j = w, w+8, ...: lanes stride the block slots
        for (int j = wid; j < it; j += kNT / 32) {
            double r = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) r += __ldcg(a.slots + (size_t)b * a.ld + j);
            r = warp_sum(r);
            if (lane == 0) a.ex.hpart[(size_t)a.g * 2 * a.ld + j] = r;
        }
        __syncthreads();
        if (tid == 0) *a.counter = 0u;
    }
}

// ---------------------------------------------------------------------------
// a9 (reorth on), exact-width passes: one launch covers basis columns
// [j0, j0 + NC) with NC a compile-time constant, so every row-vector issues
// all NC 16-byte loads at once into raw registers without predication
// (measured: 17 columns + y, u_i, u_{i-1} and the w store in ONE pass run at
// ~6.2 TB/s on B200, tools/lab/step_lab.cu). The host splits `it` columns into
// balanced passes of <= 16..17 columns; the first pass (j0 = 0) also forms the
// recurrence w = y - alpha_i v_i - beta_i v_{i-1} (mode 0) and stores it rounded.
// Same arithmetic, rounding points and reduction order as k_step.
template <typename ST, typename CT, int NC>
__global__ void __launch_bounds__(kNT, 2) k_stepw(StepArgs a, int it, int j0) {
    constexpr int VW = Vw<ST>::N;
    __shared__ CT part[kNT / 32][NC];
    __shared__ int sflag;
    if (*(volatile int *)a.st.done) return;
    if (a.gate && !*(volatile const int *)a.gate) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const ST *__restrict__ V = reinterpret_cast<const ST *>(a.V);
    const int64_t nvec = a.npad / VW;
    CT c1 = CT(0), c2 = CT(0);
    const bool form_w = (a.mode == 0 && j0 == 0);
    if (form_w) {
        double al = 0.0;
        for (int q = 0; q < a.G; ++q) al += __ldcg(a.ex.alpha_part + q);  // l.10, rank order
        const double bi = a.st.beta[it - 1];
        if (blockIdx.x == 0 && tid == 0) {
            a.st.alpha[it - 1] = al;
            double ts = *a.st.tscale;
            ts = fmax(ts, fabs(al));
            ts = fmax(ts, bi);
            *a.st.tscale = ts;
        }
        c1 = (CT)(al * a.st.scale[it - 1]);                       // alpha_i * s_i
        c2 = (it > 1 && !a.no_prev) ? (CT)(bi * a.st.scale[it - 2]) : CT(0);    // beta_i * s_{i-1}
    }
    const ST *ucur = V + (size_t)(it - 1) * a.npad;
    const ST *uprev = V + (size_t)(it > 1 ? it - 2 : 0) * a.npad;
    const ST *yv = reinterpret_cast<const ST *>(a.y);
    ST *wv = reinterpret_cast<ST *>(a.w);
    const ST *base = (a.mode == 2) ? V + (size_t)it * a.npad : wv;
    CT acc[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) acc[q] = CT(0);
    for (int64_t v = (int64_t)blockIdx.x * kNT + tid; v < nvec; v += (int64_t)gridDim.x * kNT) {
        uint4 u[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) u[q] = __ldg(reinterpret_cast<const uint4 *>(V + (size_t)(j0 + q) * a.npad + v * VW));
        CT w[VW];
        if (form_w) {
            CT yy[VW], u1[VW], u0[VW];
            vload<ST, CT>(yv + v * VW, yy);
            vload<ST, CT>(ucur + v * VW, u1);
            if (it > 1) vload<ST, CT>(uprev + v * VW, u0);
#pragma unroll
            for (int e = 0; e < VW; ++e) w[e] = yy[e] - c1 * u1[e] - (it > 1 ? c2 * u0[e] : CT(0));
            vstore_back<ST, CT>(wv + v * VW, w);  // w rounded once; dots use what was stored
        } else {
            vload<ST, CT>(base + v * VW, w);
        }
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const ST *ue = reinterpret_cast<const ST *>(&u[q]);
            CT d = CT(0);
#pragma unroll
            for (int e = 0; e < VW; ++e) d += cvt<CT>(ue[e]) * w[e];
            acc[q] += d;
        }
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const CT r = warp_sum(acc[q]);
        if (lane == 0) part[wid][q] = r;
    }
    __syncthreads();
    for (int q = tid; q < NC; q += kNT) {
        CT r = CT(0);
#pragma unroll
        for (int w8 = 0; w8 < kNT / 32; ++w8) r += part[w8][q];
        a.slots[(size_t)blockIdx.x * a.ld + j0 + q] = (double)r;
    }
    if (arrive_last(a.counter, &sflag)) {
        for (int q = wid; q < NC; q += kNT / 32) {
            double r = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) r += __ldcg(a.slots + (size_t)b * a.ld + j0 + q);
            r = warp_sum(r);
            if (lane == 0) a.ex.hpart[(size_t)a.g * 2 * a.ld + j0 + q] = r;
        }
        __syncthreads();
        if (tid == 0) *a.counter = 0u;
    }
}

// ---------------------------------------------------------------------------
// a11: correction + publish: u_{i+1} = w - sum_j h_j v_j (h_j = s_j * dot_j),
// rounded once; written to V column `it` (+ the replica slot when G > 1); norm
// partial for beta_{i+1}. in_col: -1 reads w, else reads V column in_col
// (second CGS pass corrects in place).
struct CorrArgs {
    const void *w;
    void *V;
    void *rep_slot;
    int64_t npad;
    int ld;
    double *slots;
    unsigned *counter;
    LzState st;
    Exch ex;
    int G, g, in_col;
    const int *gate;    // partial reorthogonalisation (reading Q29): run only if *gate != 0
};

// a11 shared prologue: reorth coefficients c_j = H_j s_j^2 from the dots summed over
// parts in rank order (shared memory: coef in CT, H and c in fp64), and block 0
// extends the Gram matrix (reading Q24).
template <typename CT>
__device__ __forceinline__ void corr_prologue(const CorrArgs &a, int it, double *dsm) {
    const int tid = threadIdx.x;
    CT *coef = reinterpret_cast<CT *>(dsm);
    double *hd = dsm + a.ld;   // [it] raw dots H_j (fp64)
    double *cd = hd + a.ld;    // [it] fp64 coefficients
    for (int j = tid; j < it; j += kNT) {
        double h = 0.0;
        for (int q = 0; q < a.G; ++q) h += __ldcg(a.ex.hpart + (size_t)q * 2 * a.ld + j);
        const double sj = a.st.scale[j];
        coef[j] = (CT)(h * sj * sj);
        hd[j] = h;
        cd[j] = h * sj * sj;
    }
    __syncthreads();
    if (blockIdx.x == 0 && a.st.use_gram && it < a.st.m) {
        // Gram column of the new basis vector u_{it+1} = b - sum_l coef_l u_l (b = w, or
        // the first-pass vector for CGS2) from the dots H_j = u_j . b this iteration
        // measured and the Gram of the older columns: G_{j,it} = H_j - sum_l coef_l G_{j,l}
        // (fp64; exact up to the storage rounding of u_{it+1}, reading Q24).
        // Its diagonal ||u_{it+1}||^2 is stored exactly by the next SpMV prologue.
        const int m = a.st.m;
        for (int j = tid; j < it; j += kNT) {
            double g = hd[j];
            for (int l = 0; l < it; ++l) g -= cd[l] * a.st.gram[(size_t)j * m + l];
            a.st.gram[(size_t)j * m + it] = g;
            a.st.gram[(size_t)it * m + j] = g;
        }
    }
    __syncthreads();
}

template <typename ST, typename CT>
__global__ void __launch_bounds__(kNT) k_correct(CorrArgs a, int it) {
    constexpr int VW = Vw<ST>::N;
    extern __shared__ double dsm[];  // coef[it]
    __shared__ double red_storage[kNT / 32];  // CT partials, or doubles for the final sums
    CT *red = reinterpret_cast<CT *>(red_storage);
    __shared__ int sflag;
    if (*(volatile int *)a.st.done) return;
    if (a.gate && !*(volatile const int *)a.gate) return;
    const int tid = threadIdx.x;
    CT *coef = reinterpret_cast<CT *>(dsm);
    corr_prologue<CT>(a, it, dsm);
    ST *V = reinterpret_cast<ST *>(a.V);
    const ST *src = (a.in_col < 0) ? reinterpret_cast<const ST *>(a.w) : V + (size_t)a.in_col * a.npad;
    ST *dst = V + (size_t)it * a.npad;
    const int64_t nvec = a.npad / VW;
    CT nrm = CT(0);
    // rows are walked in DESCENDING order: k_step just streamed the same basis
    // columns in ascending order, so the most recently read ones are still L2-resident
    for (int64_t vv = (int64_t)blockIdx.x * kNT + tid; vv < nvec; vv += (int64_t)gridDim.x * kNT) {
        const int64_t v = nvec - 1 - vv;
        CT acc[VW];
        vload<ST, CT>(src + v * VW, acc);
        // basis columns in blocks of 8: all loads of a block are issued before
        // the subtractions (memory-level parallelism); subtraction order stays j
        // ascending
        int j = 0;
        for (; j + 8 <= it; j += 8) {
            CT u[8][VW];
#pragma unroll
            for (int q = 0; q < 8; ++q) vload<ST, CT>(V + (size_t)(j + q) * a.npad + v * VW, u[q]);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const CT cj = coef[j + q];
#pragma unroll
                for (int e = 0; e < VW; ++e) acc[e] -= cj * u[q][e];
            }
        }
        for (; j < it; ++j) {
            CT u[VW];
            vload<ST, CT>(V + (size_t)j * a.npad + v * VW, u);
            const CT cj = coef[j];
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[e] -= cj * u[e];
        }
        vstore_back<ST, CT>(dst + v * VW, acc);
        if (a.rep_slot) vstore<ST, CT>(reinterpret_cast<ST *>(a.rep_slot) + v * VW, acc);
#pragma unroll
        for (int e = 0; e < VW; ++e) nrm += acc[e] * acc[e];
    }
    const CT tb = block_sum<CT, kNT>(nrm, red);
    if (tid == 0) a.slots[blockIdx.x] = (double)tb;
    if (arrive_last(a.counter, &sflag)) {
        const double tot = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, red_storage);
        if (tid == 0) { a.ex.norm_part[a.g] = tot; *a.counter = 0u; }
    }
}

// a11 with a compile-time column count NC = it <= kCorrMaxNC: every row-vector issues
// all NC basis loads at once into raw registers (no 8-column batches), then the
// subtractions in ascending j (the same order as k_correct).
template <typename ST, typename CT, int NC>
__global__ void __launch_bounds__(kNT) k_correctw(CorrArgs a, int it) {
    constexpr int VW = Vw<ST>::N;
    extern __shared__ double dsm[];
    __shared__ double red_storage[kNT / 32];
    CT *red = reinterpret_cast<CT *>(red_storage);
    __shared__ int sflag;
    if (*(volatile int *)a.st.done) return;
    if (a.gate && !*(volatile const int *)a.gate) return;
    const int tid = threadIdx.x;
    const CT *coef = reinterpret_cast<const CT *>(dsm);
    corr_prologue<CT>(a, it, dsm);
    ST *V = reinterpret_cast<ST *>(a.V);
    const ST *src = (a.in_col < 0) ? reinterpret_cast<const ST *>(a.w) : V + (size_t)a.in_col * a.npad;
    ST *dst = V + (size_t)it * a.npad;
    const int64_t nvec = a.npad / VW;
    CT nrm = CT(0);
    for (int64_t vv = (int64_t)blockIdx.x * kNT + tid; vv < nvec; vv += (int64_t)gridDim.x * kNT) {
        const int64_t v = nvec - 1 - vv;  // descending: the columns k_stepw just read are in L2
        uint4 u[NC];
#pragma unroll
        for (int q = 0; q < NC; ++q) u[q] = __ldg(reinterpret_cast<const uint4 *>(V + (size_t)q * a.npad + v * VW));
        CT acc[VW];
        vload<ST, CT>(src + v * VW, acc);
#pragma unroll
        for (int q = 0; q < NC; ++q) {
            const ST *ue = reinterpret_cast<const ST *>(&u[q]);
            const CT cj = coef[q];
#pragma unroll
            for (int e = 0; e < VW; ++e) acc[e] -= cj * cvt<CT>(ue[e]);
        }
        vstore_back<ST, CT>(dst + v * VW, acc);
        if (a.rep_slot) vstore<ST, CT>(reinterpret_cast<ST *>(a.rep_slot) + v * VW, acc);
#pragma unroll
        for (int e = 0; e < VW; ++e) nrm += acc[e] * acc[e];
    }
    const CT tb = block_sum<CT, kNT>(nrm, red);
    if (tid == 0) a.slots[blockIdx.x] = (double)tb;
    if (arrive_last(a.counter, &sflag)) {
        const double tot = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, red_storage);
        if (tid == 0) { a.ex.norm_part[a.g] = tot; *a.counter = 0u; }
    }
}

// ---------------------------------------------------------------------------
// a12-a13: Jacobi on T in one CTA: parallel (round-robin
// tournament) ordering of the oracle's rotations (reading Q10) with the same
// stable tangent t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta =
// (t_qq - t_pp) / (2 t_pq), evaluated division-free as
//   r = sqrt(d^2 + 4 t_pq^2), d = t_qq - t_pp, D = |d| + r,
//   c = D / sqrt(D^2 + 4 t_pq^2),  s = sgn(zeta) 2 |t_pq| / sqrt(D^2 + 4 t_pq^2)
// (c = 1/sqrt(1+t^2), s = t c with t = sgn(zeta) 2|t_pq| / D), the same
// negligibility rule (|t_pq| <= eps sqrt|t_pp t_qq| or <= eps^2 ||T||_F, tested
// squared), stop at a rotation-free sweep or max_sweeps. The M/2 rotations of
// a round are disjoint, so T <- J^T T J is applied as independent 2x2 blocks
// (pair k rows, pair l columns) and S <- S J as independent column pairs: one
// barrier-separated phase per round. Then top-K by (-|theta|, -theta) and the
// sign convention S[0,k] > 0 (reading Q12). T and S use a power-of-two leading
// dimension LD >= M (shifts instead of divisions).
struct JacArgs {
    LzState st;
    Exch ex;
    int G, m, K, max_sweeps;
    double *work;  // global workspace when T, S do not fit in shared memory
    int ld_log2;   // LD = 1 << ld_log2 >= m + (m & 1)
    int hl_log2;   // 1 << hl_log2 >= (m + (m & 1)) / 2
    // 0 -> the final solve of T_m'; 1 -> convergence check on T_i (i = m_found,
    // reading Q25): if the K selected pairs all have residual estimate
    // <= conv_tol |theta_1|, set *done = 2 (every later kernel returns at once);
    // 2 -> end of a thick-restart cycle (reading Q26): the same test, else the
    // restart data (coefR, arrow_theta, arrow_b) of the `keep` largest pairs
    int check;
    double conv_tol;
    int max_restarts;  // check == 2: no restart decision once this many restarts were done
};

// Entry (r, c) of T_mm: tridiagonal (alpha, beta), or after a thick restart
// (reading Q26) the arrowhead [[diag(theta), b], [b^T, alpha_k]] followed by the
// tridiagonal part (rows/cols >= k).
__device__ __forceinline__ double jac_t(const LzState &st, int ak, int r, int c) {
    if (r < ak || c < ak) {
        if (r == c) return st.arrow_theta[r];
        if (c == ak) return st.arrow_b[r];
        if (r == ak) return st.arrow_b[c];
        return 0.0;
    }
    if (r == c) return st.alpha[r];
    if (r - c == 1 || c - r == 1) return (r > c ? r : c) > ak ? st.beta[r > c ? r : c] : 0.0;
    return 0.0;
}

// ||T||_F of T_mm in the oracle's summation order (row-major); only the
// nonzeros are added (adding the exact zeros leaves the sum unchanged).
__device__ __forceinline__ double jac_fro(const LzState &st, int mm) {
    const int ak = *st.arrow_k;
    double f = 0.0;
    for (int r = 0; r < mm; ++r) {
        if (r < ak) {  // arrow rows: (r, r), (r, ak)
            f += st.arrow_theta[r] * st.arrow_theta[r];
            if (ak < mm) f += st.arrow_b[r] * st.arrow_b[r];
            continue;
        }
        if (r == ak && ak > 0)
            for (int c = 0; c < ak; ++c) f += st.arrow_b[c] * st.arrow_b[c];
        if (r > ak) f += st.beta[r] * st.beta[r];
        f += st.alpha[r] * st.alpha[r];
        if (r + 1 < mm) f += st.beta[r + 1] * st.beta[r + 1];
    }
    return sqrt(f);
}

// One Jacobi rotation (reading Q10): skip negligible t_pq, else the stable
// division-free (c, s) that zeroes it. Returns 1 if the rotation is applied.
__device__ __forceinline__ int jac_rotation(double apq, double app, double aqq, double fro2, double &c,
                                            double &sn) {
    const double eps = 2.220446049250313e-16;
    const double a2 = apq * apq;
    c = 1.0;
    sn = 0.0;
    if (a2 <= eps * eps * fabs(app * aqq) || a2 <= fro2) return 0;
    const double d = aqq - app;
    const bool zpos = (d == 0.0) || ((d > 0.0) == (apq > 0.0));
    const double x = d * d + 4.0 * a2;
    const double D = fabs(d) + x * rsqrt(x);
    const double ih = rsqrt(D * D + 4.0 * a2);
    c = D * ih;
    sn = (zpos ? 2.0 : -2.0) * fabs(apq) * ih;
    return 1;
}

__device__ __forceinline__ int rr_player(int pos, int round, int M) {
    if (pos == 0) return 0;
    int x = pos - 1 + round;
    if (x >= M - 1) x -= M - 1;
    return 1 + x;
}

// a13 after the sweeps: selection by (-|theta|, -theta), sign, coefficients,
// residual estimates, Ritz norms from the Gram matrix; in check mode (reading
// Q25) the stop decision instead. T, S: row-major with leading dimension 1 << LS.
__device__ void jac_finish(const JacArgs &a, const double *T, const double *S, int LS, int mm,
                           int sweeps, int conv) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const LzState &st = a.st;
    const int K = a.K;
    const int kf = K < mm ? K : mm;
    const int keep = st.keep;
    for (int c = tid; c < mm; c += nt) {
        const double tc = T[(c << LS) + c];
        st.theta_all[c] = tc;
        int rank = 0;
        for (int d = 0; d < mm; ++d) {
            const double td = T[(d << LS) + d];
            const bool before = (fabs(td) != fabs(tc)) ? (fabs(td) > fabs(tc))
                                : (td != tc) ? (td > tc) : (d < c);
            rank += before;
        }
        if (rank < kf) {
            double sg = 1.0;
            for (int j = 0; j < mm; ++j) {
                const double sj = S[(j << LS) + c];
                if (sj != 0.0) { sg = sj > 0.0 ? 1.0 : -1.0; break; }
            }
            st.evals[rank] = tc;
            for (int j = 0; j < mm; ++j) st.coefS[(size_t)j * K + rank] = sg * S[(j << LS) + c] * st.scale[j];
            st.resid[rank] = fabs(st.beta[mm] * S[((mm - 1) << LS) + c]);
            if (a.check) continue;  // norms are the final solve's business
            if (st.use_gram) {  // ||y_k||^2 = c^T G c with c_j = S[j,c] s_j (the sign cancels)
                double nrm = 0.0;
                for (int j = 0; j < mm; ++j) {
                    const double cj = S[(j << LS) + c] * st.scale[j];
                    double rowsum = 0.0;
                    for (int l = 0; l < mm; ++l) rowsum += st.gram[(size_t)j * st.m + l] * (S[(l << LS) + c] * st.scale[l]);
                    nrm += cj * rowsum;
                }
                st.rnrm2[rank] = nrm;
            }
        }
    }
    if (a.check) {
        __shared__ int s_stop;
        __syncthreads();
        if (tid == 0) {
            int ok = 0;
            if (kf == K && a.conv_tol > 0.0) {
                const double lim = a.conv_tol * fabs(st.evals[0]);
                ok = 1;
                for (int k = 0; k < K; ++k) ok &= (st.resid[k] <= lim);
                if (ok) *st.done = 2;
            }
            s_stop = ok;
        }
        __syncthreads();
        if (a.check == 2 && !s_stop) {
            // restart data (reading Q26), written only when the iteration goes on: the
            // arrowhead arrays still describe the T a stopped solve finishes with
            for (int c = tid; c < mm; c += nt) {
                const double tc = T[(c << LS) + c];
                int rank = 0;
                for (int d = 0; d < mm; ++d) {
                    const double td = T[(d << LS) + d];
                    const bool before = (fabs(td) != fabs(tc)) ? (fabs(td) > fabs(tc))
                                        : (td != tc) ? (td > tc) : (d < c);
                    rank += before;
                }
                if (rank < keep) {  // y_j = sum_l S[l][c] v_l
                    for (int l = 0; l < mm; ++l) st.coefR[(size_t)l * keep + rank] = S[(l << LS) + c] * st.scale[l];
                    st.arrow_theta[rank] = tc;
                    st.arrow_b[rank] = st.beta[mm] * S[((mm - 1) << LS) + c];
                }
            }
        }
        return;
    }
    for (int k = kf + tid; k < K; k += nt) {
        st.evals[k] = __longlong_as_double(0x7ff8000000000000ll);
        st.resid[k] = __longlong_as_double(0x7ff8000000000000ll);
    }
    if (tid == 0) {
        *st.k_found = kf;
        *st.jac_sweeps = sweeps;
        *st.jac_conv = conv;
    }
}

template <bool kSmem>
__global__ void __launch_bounds__(1024, 1) k_jacobi(JacArgs a) {
    extern __shared__ double jsm[];
    __shared__ int s_rot;
    __shared__ double s_fro;
    const int tid = threadIdx.x, nt = blockDim.x;
    const LzState &st = a.st;
    if (a.check && *(volatile int *)st.done) return;  // stopped or broke down already
    if (a.check == 2 && *st.restarts >= a.max_restarts) return;  // last cycle: the final solve follows
    const int mm = *st.m_found;
    if (tid == 0 && !*st.done) {
        double sq = 0.0;
        for (int q = 0; q < a.G; ++q) sq += __ldcg(a.ex.norm_part + q);
        st.beta[mm] = sqrt(sq);  // beta_{m'+1} (reading Q6)
    }
    __syncthreads();
    const int M = mm + (mm & 1);
    const int LS = a.ld_log2, LD = 1 << LS, HS = a.hl_log2, HD = 1 << HS;
    double *T = kSmem ? jsm : a.work;
    double *S = T + (size_t)M * LD;
    double *cs = S + (size_t)M * LD;                      // [M/2][2]
    int *pq = reinterpret_cast<int *>(cs + (size_t)M);    // [M/2][2]
    int *rot = pq + M;                                    // [M/2]
    const int ak = *st.arrow_k;
    for (int i = tid; i < M * LD; i += nt) {
        const int r = i >> LS, c = i & (LD - 1);
        const double t = (r < mm && c < mm) ? jac_t(st, ak, r, c) : 0.0;
        T[i] = t;
        S[i] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (tid == 0) s_fro = jac_fro(st, mm);
    __syncthreads();
    const double eps = 2.220446049250313e-16;
    const double fro2 = (eps * eps * s_fro) * (eps * eps * s_fro);
    int sweeps = 0, conv = (M < 2) ? 1 : 0;
    const int half = M / 2;
    while (!conv && sweeps < a.max_sweeps) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int round = 0; round < M - 1; ++round) {
            // phase A: the rotation of every pair of this round
            for (int k = tid; k < half; k += nt) {
                int p = rr_player(k, round, M), q = rr_player(M - 1 - k, round, M);
                if (p > q) { const int t = p; p = q; q = t; }
                pq[2 * k] = p;
                pq[2 * k + 1] = q;
                int doit = 0;
                double c = 1.0, sn = 0.0;
                if (q < mm) {
                    doit = jac_rotation(T[(p << LS) + q], T[(p << LS) + p], T[(q << LS) + q], fro2, c, sn);
                    if (doit) s_rot = 1;
                }
                cs[2 * k] = c;
                cs[2 * k + 1] = sn;
                rot[k] = doit;
            }
            __syncthreads();
            // phase B1: T <- J^T T J as 2x2 blocks (rows of pair k, columns of pair l).
            // Items are processed in batches of JB_: all loads of a batch first,
            // then the math, then the stores (items are disjoint within a round),
            // so a thread with many items pays one memory latency per batch
            // (matters when T, S live in global memory, m > 96)
            constexpr int JB_ = kSmem ? 1 : 4;
            const int nB1 = half << HS;
            for (int i0 = tid; i0 < nB1; i0 += nt * JB_) {
                double b[JB_][4];
                int ok[JB_];
#pragma unroll
                for (int u = 0; u < JB_; ++u) {
                    const int i = i0 + u * nt;
                    const int k = i >> HS, l = i & (HD - 1);
                    ok[u] = (i < nB1) && l < half && (rot[k] | rot[l]);
                    if (ok[u]) {
                        const int pk = pq[2 * k], qk = pq[2 * k + 1], pl = pq[2 * l], ql = pq[2 * l + 1];
                        const double *r0 = T + (pk << LS), *r1 = T + (qk << LS);
                        b[u][0] = r0[pl]; b[u][1] = r0[ql]; b[u][2] = r1[pl]; b[u][3] = r1[ql];
                    }
                }
#pragma unroll
                for (int u = 0; u < JB_; ++u) {
                    if (!ok[u]) continue;
                    const int i = i0 + u * nt;
                    const int k = i >> HS, l = i & (HD - 1);
                    const int pk = pq[2 * k], qk = pq[2 * k + 1], pl = pq[2 * l], ql = pq[2 * l + 1];
                    const double ck = cs[2 * k], sk = cs[2 * k + 1], cl = cs[2 * l], sl = cs[2 * l + 1];
                    double *r0 = T + (pk << LS), *r1 = T + (qk << LS);
                    const double e00 = cl * b[u][0] - sl * b[u][1], e01 = sl * b[u][0] + cl * b[u][1];  // T J
                    const double e10 = cl * b[u][2] - sl * b[u][3], e11 = sl * b[u][2] + cl * b[u][3];
                    const bool diag = (k == l) && rot[k];
                    r0[pl] = ck * e00 - sk * e10;                                                  // J^T .
                    r1[pl] = diag ? 0.0 : sk * e00 + ck * e10;
                    r0[ql] = diag ? 0.0 : ck * e01 - sk * e11;
                    r1[ql] = sk * e01 + ck * e11;
                }
            }
            // phase B2: S <- S J (columns p, q), row r, same batching
            const int nB2 = half << LS;
            for (int i0 = tid; i0 < nB2; i0 += nt * JB_) {
                double sv[JB_][2];
                int ok[JB_];
#pragma unroll
                for (int u = 0; u < JB_; ++u) {
                    const int i = i0 + u * nt;
                    const int k = i >> LS, r = i & (LD - 1);
                    ok[u] = (i < nB2) && r < mm && rot[k];
                    if (ok[u]) {
                        const double *Sr = S + (r << LS);
                        sv[u][0] = Sr[pq[2 * k]];
                        sv[u][1] = Sr[pq[2 * k + 1]];
                    }
                }
#pragma unroll
                for (int u = 0; u < JB_; ++u) {
                    if (!ok[u]) continue;
                    const int i = i0 + u * nt;
                    const int k = i >> LS, r = i & (LD - 1);
                    const double c = cs[2 * k], sn = cs[2 * k + 1];
                    double *Sr = S + (r << LS);
                    Sr[pq[2 * k]] = c * sv[u][0] - sn * sv[u][1];
                    Sr[pq[2 * k + 1]] = sn * sv[u][0] + c * sv[u][1];
                }
            }
            __syncthreads();
        }
        ++sweeps;
        conv = !s_rot;
        __syncthreads();
    }
    jac_finish(a, T, S, LS, mm, sweeps, conv);
}

// ---------------------------------------------------------------------------
// a12 for large m (T and S of one part do not fit one SM's shared memory): the
// same round-robin rounds and rotation formula as k_jacobi (reading Q10), on a
// thread-block cluster. CTA b owns rows [bR, (b+1)R) of T (two buffers: the row
// op of a round writes the other one) and of S, in its shared memory. Per round:
//  (A) every CTA derives all M/2 rotations from t_pp, t_qq, t_pq (distributed
//      shared memory reads; identical results in every CTA, so the stop test
//      needs no exchange);
//  (B) column op T <- T J and S <- S J on its own rows; cluster barrier;
//  (C) row op T <- J^T T into the other buffer, the partner row read remotely;
//      the rotated pair's (p, q) entries set to exact zero; cluster barrier.
// Then T's diagonal and S go to the global workspace and CTA 0 finishes.
constexpr int kJacClNT = 1024;

__global__ void __launch_bounds__(kJacClNT, 1) k_jacobi_cl(JacArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ double jsm[];
    __shared__ int s_rot;
    __shared__ double s_fro;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int br = (int)cl.block_rank(), CL = (int)cl.num_blocks();
    const LzState &st = a.st;
    if (a.check && *(volatile int *)st.done) return;  // same value in every CTA
    if (a.check == 2 && *st.restarts >= a.max_restarts) return;
    const int mm = *st.m_found;
    if (br == 0 && tid == 0 && !*st.done) {
        double sq = 0.0;
        for (int q = 0; q < a.G; ++q) sq += __ldcg(a.ex.norm_part + q);
        st.beta[mm] = sqrt(sq);  // beta_{m'+1} (reading Q6)
    }
    const int M = mm + (mm & 1), half = M / 2;
    const int R = (M + CL - 1) / CL, LDc = M;
    const int r0 = br * R;
    const int nloc = (r0 >= M) ? 0 : ((M - r0) < R ? (M - r0) : R);
    double *T0 = jsm, *T1 = T0 + (size_t)R * LDc, *Sl = T1 + (size_t)R * LDc;
    double *cs = Sl + (size_t)R * LDc;                  // [half][2]
    int *pq = reinterpret_cast<int *>(cs + 2 * half);  // [half][2]
    int *rot = pq + 2 * half;                          // [half]
    int *prow = rot + half;                            // [M]: 2 k + (row is the q of pair k)
    const int ak = *st.arrow_k;
    for (int i = tid; i < nloc * LDc; i += nt) {
        const int rl = i / LDc, c = i - rl * LDc, r = r0 + rl;
        const double t = (r < mm && c < mm) ? jac_t(st, ak, r, c) : 0.0;
        T0[i] = t;
        Sl[i] = (r == c) ? 1.0 : 0.0;
    }
    if (tid == 0) s_fro = jac_fro(st, mm);
    __syncthreads();
    const double eps = 2.220446049250313e-16;
    const double fro2 = (eps * eps * s_fro) * (eps * eps * s_fro);
    cl.sync();  // every CTA's rows are initialised before the first remote read
    int sweeps = 0, conv = (M < 2) ? 1 : 0, cur = 0;
    while (!conv && sweeps < a.max_sweeps) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int round = 0; round < M - 1; ++round) {
            double *Tc = cur ? T1 : T0, *Tn = cur ? T0 : T1;
            // (A) rotations of this round
            for (int k = tid; k < half; k += nt) {
                int p = rr_player(k, round, M), q = rr_player(M - 1 - k, round, M);
                if (p > q) { const int t = p; p = q; q = t; }
                pq[2 * k] = p;
                pq[2 * k + 1] = q;
                prow[p] = 2 * k;
                prow[q] = 2 * k + 1;
                int doit = 0;
                double c = 1.0, sn = 0.0;
                if (q < mm) {
                    const double *Rp = cl.map_shared_rank(Tc, p / R) + (size_t)(p % R) * LDc;
                    const double *Rq = cl.map_shared_rank(Tc, q / R) + (size_t)(q % R) * LDc;
                    doit = jac_rotation(Rp[q], Rp[p], Rq[q], fro2, c, sn);
                    if (doit) s_rot = 1;
                }
                cs[2 * k] = c;
                cs[2 * k + 1] = sn;
                rot[k] = doit;
            }
            __syncthreads();
            // (B) T <- T J, S <- S J on the own rows
            for (int i = tid; i < nloc * half; i += nt) {
                const int rl = i / half, k = i - rl * half;
                if (!rot[k]) continue;
                const int p = pq[2 * k], q = pq[2 * k + 1];
                const double c = cs[2 * k], sn = cs[2 * k + 1];
                double *tr = Tc + (size_t)rl * LDc, *sr = Sl + (size_t)rl * LDc;
                const double tp = tr[p], tq = tr[q], sp = sr[p], sq = sr[q];
                tr[p] = c * tp - sn * tq;
                tr[q] = sn * tp + c * tq;
                sr[p] = c * sp - sn * sq;
                sr[q] = sn * sp + c * sq;
            }
            cl.sync();
            // (C) T <- J^T T into the other buffer (batching several remote loads per
            // thread measured slower: register-limited at 1024 threads)
            for (int i = tid; i < nloc * M; i += nt) {
                const int rl = i / M, col = i - rl * M, r = r0 + rl;
                const int pk = prow[r], k = pk >> 1, isq = pk & 1;
                double v = Tc[(size_t)rl * LDc + col];
                if (rot[k]) {
                    const int partner = pq[2 * k + (isq ^ 1)];
                    const double w = cl.map_shared_rank(Tc, partner / R)[(size_t)(partner % R) * LDc + col];
                    const double c = cs[2 * k], sn = cs[2 * k + 1];
                    v = isq ? (sn * w + c * v) : (c * v - sn * w);
                    if (col == partner) v = 0.0;  // the annihilated t_pq, t_qp
                }
                Tn[(size_t)rl * LDc + col] = v;
            }
            cl.sync();
            cur ^= 1;
        }
        ++sweeps;
        conv = !s_rot;
        __syncthreads();
    }
    // results to the global workspace (T diagonal, S rows), CTA 0 finishes
    const int LS = a.ld_log2;
    double *Tg = a.work, *Sg = a.work + ((size_t)M << LS);
    const double *Tf = cur ? T1 : T0;
    for (int i = tid; i < nloc * M; i += nt) {
        const int rl = i / M, col = i - rl * M, r = r0 + rl;
        Sg[((size_t)r << LS) + col] = Sl[(size_t)rl * LDc + col];
        if (col == r) Tg[((size_t)r << LS) + r] = Tf[(size_t)rl * LDc + col];
    }
    __threadfence();
    cl.sync();
    if (br != 0) return;
    jac_finish(a, Tg, Sg, LS, mm, sweeps, conv);
}

// ---------------------------------------------------------------------------
// a14: Ritz projection y_k = sum_j S[j,k] v_j ("the eigenvectors of
// M are given by 𝒱V"), fp64 accumulation, then y_k / ||y_k|| (reading Q12).
// Two streaming passes over the stored basis; no fp64 Y is materialised:
//   pass 0: recompute y_k row by row, per-block partials of ||y_k||^2 ->
//           ex.ritz_part[g][k] (last-arriving block per output group, fixed order)
//   pass 1: recompute y_k, scale by 1/||y_k|| (norms summed over parts in rank
//           order) and store once, in the output dtype, in position order
//           blocked by output group (yt[g][p][q], k = g KB + q; coalesced
//           stores); k_unperm then writes the caller's buffer in original row
//           order (one 32/64-byte sector per group per row).
// Thread = VW consecutive rows (one 16-byte load per basis column) x KB outputs;
// block b = (row range b / ngroups, output group b % ngroups). coefS holds the sign
// fix and the deferred normalisation s_j.
struct RitzArgs {
    const void *V;
    int64_t npad, nrows;
    int K, G, g;
    double *slots;            // [gridDim.x][K]
    unsigned *counter;        // [ceil(K / KB)]
    LzState st;
    Exch ex;
    void *const *out_ptr;     // device param: output base (pass 1 writes only if non-NULL)
    const int *out_dtype;     // device param: 0 f64, 1 f32
    void *yt;                 // [ceil(K/KB)][npad][KB] Ritz vectors in position order, output dtype
};

template <typename ST, typename CT, int KB, int pass>
__global__ void __launch_bounds__(kNT, 2) k_ritz(RitzArgs a) {
    constexpr int VW = Vw<ST>::N;
    extern __shared__ double rsm[];  // coef[m'][KB]
    __shared__ CT part[kNT / 32][KB];
    __shared__ double inv[KB];
    __shared__ int sflag;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int mm = *a.st.m_found, kf = *a.st.k_found, K = a.K;
    // output group fastest: the ngroups blocks of one row range run together and
    // share the basis reads through L2 (DRAM reads V once per pass)
    const int ngroups = (K + KB - 1) / KB;
    const int grp = (int)(blockIdx.x % (unsigned)ngroups);
    const int rblk = (int)(blockIdx.x / (unsigned)ngroups), nrblk = (int)(gridDim.x / (unsigned)ngroups);
    const int k0 = grp * KB;
    if (k0 >= kf) return;
    void *out = nullptr;
    int dt = 0;
    if (pass == 1) {
        out = *a.out_ptr;
        if (!out) return;
        dt = *a.out_dtype;
    }
    CT *coef = reinterpret_cast<CT *>(rsm);
    for (int i = tid; i < mm * KB; i += kNT) {
        const int j = i / KB, q = i - j * KB;
        coef[i] = (k0 + q < kf) ? (CT)a.st.coefS[(size_t)j * K + k0 + q] : CT(0);
    }
    if (pass == 1 && tid < KB) {
        double s = 0.0;
        if (a.st.use_gram) s = (k0 + tid < kf) ? a.st.rnrm2[k0 + tid] : 1.0;
        else
            for (int q = 0; q < a.G; ++q) s += __ldcg(a.ex.ritz_part + (size_t)q * K + k0 + tid);
        inv[tid] = (k0 + tid < kf) ? 1.0 / sqrt(s) : 0.0;
    }
    __syncthreads();
    const ST *V = reinterpret_cast<const ST *>(a.V);
    const int64_t nvec = (a.nrows + VW - 1) / VW;
    CT nrm[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) nrm[q] = CT(0);
    for (int64_t v = (int64_t)rblk * kNT + tid; v < nvec; v += (int64_t)nrblk * kNT) {
        CT acc[VW][KB];
#pragma unroll
        for (int e = 0; e < VW; ++e)
#pragma unroll
            for (int q = 0; q < KB; ++q) acc[e][q] = CT(0);
        // basis columns 4 at a time: the 4 loads are in flight together (raw
        // registers), then 4 x VW x KB fp64 FMAs; coefficient pairs via 16-byte
        // shared-memory broadcasts
        constexpr int JU = 4;
        for (int j0 = 0; j0 < mm; j0 += JU) {
            int4 raw[JU];
#pragma unroll
            for (int t = 0; t < JU; ++t)
                raw[t] = (j0 + t < mm) ? ld_stream(reinterpret_cast<const int4 *>(V + (size_t)(j0 + t) * a.npad + v * VW))
                                       : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int t = 0; t < JU; ++t) {
                if (j0 + t >= mm) break;
                const ST *ue = reinterpret_cast<const ST *>(&raw[t]);
                CT u[VW];
#pragma unroll
                for (int e = 0; e < VW; ++e) u[e] = cvt<CT>(ue[e]);
                const CT *cj = coef + (j0 + t) * KB;
#pragma unroll
                for (int q = 0; q < KB; ++q) {
                    const CT c = cj[q];
#pragma unroll
                    for (int e = 0; e < VW; ++e) acc[e][q] += c * u[e];
                }
            }
        }
        if (pass == 0) {
#pragma unroll
            for (int q = 0; q < KB; ++q)
#pragma unroll
                for (int e = 0; e < VW; ++e) nrm[q] += acc[e][q] * acc[e][q];
        } else {
            // yt layout [group][position][KB]: this thread's VW rows x KB outputs are
            // one contiguous block and consecutive lanes own consecutive blocks, so
            // the stores are fully coalesced 16-byte vectors
            const size_t o = ((size_t)grp * a.npad + (size_t)v * VW) * KB;
            if (dt == 0) {
                double *dst = reinterpret_cast<double *>(a.yt) + o;
#pragma unroll
                for (int e = 0; e < VW; ++e)
#pragma unroll
                    for (int q = 0; q < KB; q += 2)
                        __stcs(reinterpret_cast<double2 *>(dst + e * KB + q),
                               make_double2((double)acc[e][q] * inv[q], (double)acc[e][q + 1] * inv[q + 1]));
            } else {
                float *dst = reinterpret_cast<float *>(a.yt) + o;
#pragma unroll
                for (int e = 0; e < VW; ++e)
#pragma unroll
                    for (int q = 0; q < KB; q += 4)
                        __stcs(reinterpret_cast<float4 *>(dst + e * KB + q),
                               make_float4((float)(acc[e][q] * inv[q]), (float)(acc[e][q + 1] * inv[q + 1]),
                                           (float)(acc[e][q + 2] * inv[q + 2]), (float)(acc[e][q + 3] * inv[q + 3])));
            }
        }
    }
    if constexpr (pass == 1) {
        return;
    } else {
#pragma unroll
    for (int q = 0; q < KB; ++q) {
        const CT rr = warp_sum(nrm[q]);
        if (lane == 0) part[wid][q] = rr;
    }
    __syncthreads();
    if (tid < KB && k0 + tid < kf) {
        CT rr = CT(0);
#pragma unroll
        for (int w8 = 0; w8 < kNT / 32; ++w8) rr += part[w8][tid];
        a.slots[(size_t)rblk * K + k0 + tid] = (double)rr;
    }
    if (arrive_last_n(a.counter + grp, (unsigned)nrblk, &sflag)) {
        for (int q = wid; q < KB; q += kNT / 32) {
            if (k0 + q >= kf) break;
            double rr = 0.0;
            for (int b = lane; b < nrblk; b += 32) rr += __ldcg(a.slots + (size_t)b * K + k0 + q);
            rr = warp_sum(rr);
            if (lane == 0) a.ex.ritz_part[(size_t)a.g * K + k0 + q] = rr;
        }
        __syncthreads();
        if (tid == 0) a.counter[grp] = 0u;
    }
    }
}

// a14 output pass on the fp64 tensor-core path (mma.sync m8n8k4 f64, DMMA): the same
// projection Y = V_stored C (C = coefS: S_K diag(s), sign-fixed) and scaling by
// 1/||y_k|| as k_ritz pass 1, for compute dtype f64. A warp owns 32 positions x 8 TN
// outputs: per step of 4 basis columns it loads one f32/f64 basis element per position
// tile (A fragments, converted to f64) and one coefficient per output tile from shared
// memory (B fragments), and issues TM x TN DMMAs; accumulators stay in registers. The
// coefficients of the block's output group are staged once in shared memory
// [mm rounded up to 4][8 TN]. Writes yt[group][position][8] like k_ritz pass 1.
__device__ __forceinline__ void dmma_8x8x4(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
#ifndef TOPK_RITZ_TM
#define TOPK_RITZ_TM 8
#endif
constexpr int kRitzTM = TOPK_RITZ_TM;  // position tiles of 8 per warp (dev build variant)
template <typename ST, int TN>
__global__ void __launch_bounds__(kNT, 2) k_ritz_mma(RitzArgs a) {
    static_assert(kRitzKB == 8, "yt groups of 8 outputs");
    constexpr int TM = TN >= 4 ? 4 : kRitzTM;  // 8 x 4 position tiles spill at 4 output tiles
    extern __shared__ double csm[];  // coef [mm4][8 TN], then inv [8 TN]
    constexpr int NO = 8 * TN;
    const int tid = threadIdx.x, lane = tid & 31;
    const int mm = *a.st.m_found, kf = *a.st.k_found, K = a.K;
    const int nog = (K + NO - 1) / NO;
    const int og = (int)(blockIdx.x % (unsigned)nog);
    const int rblk = (int)(blockIdx.x / (unsigned)nog), nrblk = (int)(gridDim.x / (unsigned)nog);
    const int k0 = og * NO;
    if (k0 >= kf) return;
    void *out = *a.out_ptr;
    if (!out) return;
    const int dt = *a.out_dtype;
    const int mm4 = (mm + 3) & ~3;
    double *coef = csm;
    double *inv = csm + (size_t)mm4 * NO;
    for (int i = tid; i < mm4 * NO; i += kNT) {
        const int j = i / NO, q = i - j * NO;
        coef[i] = (j < mm && k0 + q < kf) ? a.st.coefS[(size_t)j * K + k0 + q] : 0.0;
    }
    if (tid < NO) {
        double sq = 0.0;
        if (a.st.use_gram) sq = (k0 + tid < kf) ? a.st.rnrm2[k0 + tid] : 1.0;
        else
            for (int q = 0; q < a.G; ++q) sq += __ldcg(a.ex.ritz_part + (size_t)q * K + k0 + tid);
        inv[tid] = (k0 + tid < kf) ? 1.0 / sqrt(sq) : 0.0;
    }
    __syncthreads();
    const ST *V = reinterpret_cast<const ST *>(a.V);
    const int r = lane >> 2, c = lane & 3;  // fragment row / column of this lane
    const int64_t ntile = a.npad / (8 * TM);
    const int warp = (int)(rblk * (kNT / 32) + (tid >> 5)), nwarp = nrblk * (kNT / 32);
    for (int64_t t = warp; t < ntile; t += nwarp) {
        const int64_t p0 = t * 8 * TM;
        double acc[TM][TN][2];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int n = 0; n < TN; ++n) acc[i][n][0] = acc[i][n][1] = 0.0;
        // A fragments one step ahead: the next 4 basis columns' loads are in flight
        // while this step's DMMAs run
        ST araw[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i)
            araw[i] = (c < mm) ? V[(size_t)c * a.npad + p0 + 8 * i + r] : ST(0);
        for (int j0 = 0; j0 < mm4; j0 += 4) {
            double af[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i) af[i] = cvt<double>(araw[i]);
            const int jn = j0 + 4 + c;
#pragma unroll
            for (int i = 0; i < TM; ++i)
                araw[i] = (jn < mm) ? V[(size_t)jn * a.npad + p0 + 8 * i + r] : ST(0);
            double bf[TN];
#pragma unroll
            for (int n = 0; n < TN; ++n) bf[n] = coef[(j0 + c) * NO + 8 * n + r];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int n = 0; n < TN; ++n) dmma_8x8x4(acc[i][n][0], acc[i][n][1], af[i], bf[n]);
        }
        // D fragment: lane holds rows r, columns 2c, 2c + 1 of each 8 x 8 tile
#pragma unroll
        for (int i = 0; i < TM; ++i) {
            const int64_t p = p0 + 8 * i + r;
#pragma unroll
            for (int n = 0; n < TN; ++n) {
                if ((og * TN + n) * 8 >= K) break;  // groups past ceil(K / 8): not in yt
                const int kk = 8 * n + 2 * c;
                const double y0 = acc[i][n][0] * inv[kk], y1 = acc[i][n][1] * inv[kk + 1];
                const size_t o = ((size_t)(og * TN + n) * a.npad + (size_t)p) * kRitzKB + 2 * c;
                if (dt == 0) __stcs(reinterpret_cast<double2 *>(reinterpret_cast<double *>(a.yt) + o), make_double2(y0, y1));
                else __stcs(reinterpret_cast<float2 *>(reinterpret_cast<float *>(a.yt) + o), make_float2((float)y0, (float)y1));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Thick restart (reading Q26; not in the paper):
// Y_j = sum_l coefR[l][j] u_l (coefR = S_J diag(s), the kept Ritz vectors of the
// cycle's T), rounded to the storage dtype into the scratch columns, with the
// squared norm of each stored y_j (fp64 partials, last block per output group
// sums them in block order -> ex.rst_part[g][j]). One pass over the basis per
// group of KB kept vectors.
struct RestartArgs {
    void *V;             // basis (mm + 1 columns used)
    void *Vs;            // scratch: keep columns of npad
    int64_t npad;
    int keep, G, g, mm;
    double *slots;       // [gridDim.x][KB]
    unsigned *counter;   // [ceil(keep / KB)]
    LzState st;
    Exch ex;
};

template <typename ST, typename CT, int KB>
__global__ void __launch_bounds__(kNT, 2) k_restart_proj(RestartArgs a) {
    constexpr int VW = Vw<ST>::N;
    extern __shared__ double rsm[];  // coef[mm][KB]
    __shared__ CT part[kNT / 32][KB];
    __shared__ int sflag;
    if (*(volatile int *)a.st.done) return;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int mm = a.mm, keep = a.keep;
    const int ngroups = (keep + KB - 1) / KB;
    const int grp = (int)(blockIdx.x % (unsigned)ngroups);
    const int rblk = (int)(blockIdx.x / (unsigned)ngroups), nrblk = (int)(gridDim.x / (unsigned)ngroups);
    const int k0 = grp * KB;
    CT *coef = reinterpret_cast<CT *>(rsm);
    for (int i = tid; i < mm * KB; i += kNT) {
        const int j = i / KB, q = i - j * KB;
        coef[i] = (k0 + q < keep) ? (CT)a.st.coefR[(size_t)j * keep + k0 + q] : CT(0);
    }
    __syncthreads();
    const ST *V = reinterpret_cast<const ST *>(a.V);
    ST *Vs = reinterpret_cast<ST *>(a.Vs);
    const int64_t nvec = a.npad / VW;
    CT nrm[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) nrm[q] = CT(0);
    for (int64_t v = (int64_t)rblk * kNT + tid; v < nvec; v += (int64_t)nrblk * kNT) {
        CT acc[VW][KB];
#pragma unroll
        for (int e = 0; e < VW; ++e)
#pragma unroll
            for (int q = 0; q < KB; ++q) acc[e][q] = CT(0);
        constexpr int JU = 4;
        for (int j0 = 0; j0 < mm; j0 += JU) {
            int4 raw[JU];
#pragma unroll
            for (int t = 0; t < JU; ++t)
                raw[t] = (j0 + t < mm) ? ld_stream(reinterpret_cast<const int4 *>(V + (size_t)(j0 + t) * a.npad + v * VW))
                                       : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int t = 0; t < JU; ++t) {
                if (j0 + t >= mm) break;
                const ST *ue = reinterpret_cast<const ST *>(&raw[t]);
                CT u[VW];
#pragma unroll
                for (int e = 0; e < VW; ++e) u[e] = cvt<CT>(ue[e]);
                const CT *cj = coef + (j0 + t) * KB;
#pragma unroll
                for (int q = 0; q < KB; ++q) {
                    const CT c = cj[q];
#pragma unroll
                    for (int e = 0; e < VW; ++e) acc[e][q] += c * u[e];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < KB; ++q) {
            if (k0 + q >= keep) break;
            CT yq[VW];
#pragma unroll
            for (int e = 0; e < VW; ++e) yq[e] = acc[e][q];
            vstore_back<ST, CT>(Vs + (size_t)(k0 + q) * a.npad + v * VW, yq);  // rounded once
#pragma unroll
            for (int e = 0; e < VW; ++e) nrm[q] += yq[e] * yq[e];             // norm of what is stored
        }
    }
#pragma unroll
    for (int q = 0; q < KB; ++q) {
        const CT rr = warp_sum(nrm[q]);
        if (lane == 0) part[wid][q] = rr;
    }
    __syncthreads();
    if (tid < KB) {
        CT rr = CT(0);
#pragma unroll
        for (int w8 = 0; w8 < kNT / 32; ++w8) rr += part[w8][tid];
        a.slots[(size_t)blockIdx.x * KB + tid] = (double)rr;
    }
    if (arrive_last_n(a.counter + grp, (unsigned)nrblk, &sflag)) {
        if (tid < KB && k0 + tid < keep) {
            double rr = 0.0;
            for (int b = 0; b < nrblk; ++b) rr += __ldcg(a.slots + ((size_t)b * ngroups + grp) * KB + tid);
            a.ex.rst_part[(size_t)a.g * keep + k0 + tid] = rr;
        }
        __syncthreads();
        if (tid == 0) a.counter[grp] = 0u;
    }
}

// Restart bookkeeping: V[0..keep) <- the stored Ritz vectors, V[keep] <- u_{m+1}
// (the cycle's last, unnormalised residual vector; its norm is still in the norm
// partials, so the next SpMV prologue sets beta and s for it), s_j = 1/||y_j||
// (norm partials summed over parts in rank order), the arrowhead size k.
template <typename ST>
__global__ void __launch_bounds__(kNT) k_restart_copy(RestartArgs a) {
    if (*(volatile int *)a.st.done) return;
    const int keep = a.keep;
    if (blockIdx.x == 0 && threadIdx.x < keep) {
        const int j = threadIdx.x;
        double s = 0.0;
        for (int q = 0; q < a.G; ++q) s += __ldcg(a.ex.rst_part + (size_t)q * keep + j);
        a.st.scale[j] = 1.0 / sqrt(s);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.st.arrow_k = keep;
        *a.st.m_found = keep;
        *a.st.restarts += 1;
    }
    // 16-byte words (n_pad is a multiple of 64 rows)
    const int64_t nw = a.npad * (int64_t)sizeof(ST) / 16;
    const uint4 *Vs = reinterpret_cast<const uint4 *>(a.Vs);
    uint4 *V = reinterpret_cast<uint4 *>(a.V);
    const int64_t tot = nw * (keep + 1);
    for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < tot; i += (int64_t)gridDim.x * kNT) {
        const int64_t j = i / nw, w = i - j * nw;
        V[j * nw + w] = (j < keep) ? Vs[j * nw + w] : V[(int64_t)a.mm * nw + w];
    }
}

// ---------------------------------------------------------------------------
// a4 on the device: the physical SpMV arrays from the part's canonical CSR slice
// (uploaded as is, values already rounded to the value storage dtype), with the
// host rule of build_part (host_prep.cpp): position p holds original part row
// perm[p]; entry e of a big row goes to rowptr_deg[p] + e, entry e of SELL slice
// row i to base + 32 e + i, padding (column 0, value 0); columns through colmap.
// MODE 0: every entry; MODE 1: the own-slot entries (device column / n_pad == g, the
// first pass of the two-pass SpMV); MODE 2: the others (the final pass).
template <int MODE> __device__ __forceinline__ bool pass_keeps(int32_t c, int64_t npad, int g) {
    if constexpr (MODE == 0) return true;
    const bool own = (int64_t)c / npad == (int64_t)g;
    return MODE == 1 ? own : !own;
}

// big rows: warp per row; the j-th kept entry (input order) goes to dbig[p] + j
template <typename VT, int MODE>
__global__ void __launch_bounds__(256) k_layout_big(const int64_t *srp, const int32_t *scol, const VT *sval,
                                                    const int32_t *perm, const int64_t *dbig, const int32_t *colmap,
                                                    int nbig, int64_t nphys, int64_t npad, int g, int32_t *pcol,
                                                    VT *pval) {
    (void)nphys;
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = w; p < nbig; p += nw) {
        const int r = perm[p];
        const int64_t k0 = srp[r], len = srp[r + 1] - k0, d0 = dbig[p];
        int64_t written = 0;
        for (int64_t e0 = 0; e0 < len; e0 += 32) {
            const int64_t e = e0 + lane;
            int32_t c = 0;
            bool keep = false;
            if (e < len) {
                c = colmap[scol[k0 + e]];
                keep = pass_keeps<MODE>(c, npad, g);
            }
            const unsigned msk = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int64_t d = d0 + written + __popc(msk & ((1u << lane) - 1u));
                TOPK_DCHECK(d < nphys && d < dbig[p + 1], "big-row scatter destination");
                pcol[d] = c;
                pval[d] = sval[k0 + e];
            }
            written += __popc(msk);
        }
    }
}

// big rows, single pass (MODE 0: every entry kept, so entry j of row p goes to
// dbig[p] + j = the logical offset): warp per SpMV chunk (<= kChunkNnz entries), so a
// hub row of ~10^5 entries is spread over many warps instead of one (k_layout_big's
// warp per row took 3.5 ms on C3 for its longest row alone)
template <typename VT>
__global__ void __launch_bounds__(256) k_layout_big_chunks(const int64_t *srp, const int32_t *scol, const VT *sval,
                                                           const int32_t *perm, const int64_t *drp, const Chunk *chunks,
                                                           int nchunks, const int32_t *colmap, int64_t nphys, int32_t *pcol,
                                                           VT *pval) {
    (void)nphys;
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t ci = w; ci < nchunks; ci += nw) {
        const Chunk C = chunks[ci];
        const int64_t src0 = srp[perm[C.row]] + (C.z0 - drp[C.row]);
        constexpr int U = 8;
        for (int e0 = 0; e0 < C.cnt; e0 += 32 * U) {
            int32_t c[U];
            VT v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + 32 * u + lane;
                c[u] = e < C.cnt ? scol[src0 + e] : 0;
                v[u] = e < C.cnt ? sval[src0 + e] : VT(0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int e = e0 + 32 * u + lane;
                if (e < C.cnt) {
                    TOPK_DCHECK(C.z0 + e < nphys && C.z0 + e >= drp[C.row] && C.z0 + e < drp[C.row + 1],
                                "big-row chunk scatter destination");
                    pcol[C.z0 + e] = colmap[c[u]];
                    pval[C.z0 + e] = v[u];
                }
            }
        }
    }
}

// SELL slices: thread per slice row; the j-th kept entry to base + 32 j + i, then padding
template <typename VT, int MODE>
__global__ void __launch_bounds__(256) k_layout_sell(const int64_t *srp, const int32_t *scol, const VT *sval,
                                                     const int32_t *perm, const int64_t *drp, const int32_t *colmap,
                                                     const longlong2 *sell, int64_t nbig, int64_t nne, int64_t nsl,
                                                     int64_t nphys, int64_t npad, int g, int32_t *pcol, VT *pval) {
    (void)nphys;
    const int64_t tot = 32 * nsl;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t sl = i >> 5, lane = i & 31, p = nbig + i;
        const longlong2 S = sell[sl];
        int64_t len = 0, k0 = 0;
        if (p < nne) {
            len = drp[p + 1] - drp[p];
            k0 = srp[perm[p]];
        }
        TOPK_DCHECK(S.x + 32 * S.y <= nphys, "SELL slice bounds");
        int64_t j = 0;
        for (int64_t e = 0; e < len; ++e) {
            const int32_t c = colmap[scol[k0 + e]];
            if (!pass_keeps<MODE>(c, npad, g)) continue;
            TOPK_DCHECK(j < S.y, "SELL row longer than its slice");
            const int64_t d = S.x + 32 * j + lane;
            pcol[d] = c;
            pval[d] = sval[k0 + e];
            ++j;
        }
        for (; j < S.y; ++j) {
            const int64_t d = S.x + 32 * j + lane;
            pcol[d] = 0;
            pval[d] = VT(0);
        }
    }
}

// own-slot entries per position (the first pass's degrees), warp per row
__global__ void __launch_bounds__(256) k_own_count(const int64_t *srp, const int32_t *scol, const int32_t *perm,
                                                   const int32_t *colmap, int64_t nne, int64_t npad, int g,
                                                   int32_t *cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = w; p < nne; p += nw) {
        const int r = perm[p];
        const int64_t k0 = srp[r], len = srp[r + 1] - k0;
        int c = 0;
        for (int64_t e = lane; e < len; e += 32) c += pass_keeps<1>(colmap[scol[k0 + e]], npad, g);
        c = warp_sum(c);
        if (lane == 0) cnt[p] = c;
    }
}

// ---------------------------------------------------------------------------
// Halo exchange (reading Q27). x_g = [own slot |
// remote entries grouped by owner]; EL is the storage element as raw bits.
//  k_halo_pull (parts on one device): x_g[n_pad + t] = x_{q_t}[pos_t]
//  k_halo_pack (one process per GPU): send[t] = x_g[send_pos[t]] (then NCCL send/recv)
template <typename EL>
__global__ void __launch_bounds__(256) k_halo_pull(EL *xg, int64_t npad, int64_t nhalo, const int32_t *hq,
                                                   const int32_t *hpos, const EL *const *src) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nhalo; t += (int64_t)gridDim.x * blockDim.x)
        xg[npad + t] = src[hq[t]][hpos[t]];
}
template <typename EL>
__global__ void __launch_bounds__(256) k_halo_pack(const EL *xg, int64_t nsend, const int32_t *spos, EL *sendbuf) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nsend; t += (int64_t)gridDim.x * blockDim.x)
        sendbuf[t] = xg[spos[t]];
}

// Thick-restart loop condition of the CUDA graph's WHILE node (reading Q26): one more
// restart cycle while the iteration has not stopped and fewer than R restarts are done.
__global__ void k_restart_cond(cudaGraphConditionalHandle ch, const int *done, const int *restarts, int R) {
    if (threadIdx.x == 0)
        cudaGraphSetConditional(ch, (*(volatile const int *)done == 0 && *(volatile const int *)restarts < R) ? 1u : 0u);
}

// ---------------------------------------------------------------------------
// Partial reorthogonalisation (reading Q29; Simon 1984):
// after the three-term step of iteration `it`, Simon's recurrence estimates the
// orthogonality w_{it+1,k} of the new vector against v_1..v_{it-1} (the oracle's order
// of operations, no contraction); the pass (the CGS2 second-pass kernels on V[:, it])
// runs when max |w| > sqrt(eps), and on the next vector too. Rows of w rotate in W[3].
struct ProArgs {
    LzState st;
    Exch ex;
    int G;
    double eps, psi;   // storage unit roundoff; w_{j+1,j} = psi = eps sqrt(n)
    double *W;         // [3][m + 2]
    int *gate, *force, *count;
};

__global__ void __launch_bounds__(256) k_pro(ProArgs a, int it) {
    __shared__ double s_b, s_max[8];
    const int tid = threadIdx.x;
    if (*(volatile int *)a.st.done) return;
    const int ld = a.st.m + 2;
    double *prev = a.W + (size_t)((it + 2) % 3) * ld, *cur = a.W + (size_t)(it % 3) * ld;
    double *nw = a.W + (size_t)((it + 1) % 3) * ld;
    if (it == 1) {
        for (int k = tid; k < ld; k += blockDim.x) { prev[k] = 0.0; cur[k] = 0.0; }
        __syncthreads();
        if (tid == 0) { cur[1] = 1.0; *a.force = 0; *a.count = 0; }
    }
    if (tid == 0) {
        double sq = 0.0;
        for (int q = 0; q < a.G; ++q) sq += __ldcg(a.ex.norm_part + q);
        s_b = sqrt(sq);  // beta_{it+1} before any reorthogonalisation
    }
    __syncthreads();
    const double b = s_b, ai = a.st.alpha[it - 1], bi = a.st.beta[it - 1];
    const double *al = a.st.alpha, *be = a.st.beta;
    double mx = 0.0;
    for (int k = 1 + tid; k < it; k += blockDim.x) {
        double t = __dadd_rn(__dmul_rn(be[k], cur[k + 1]), __dmul_rn(__dsub_rn(al[k - 1], ai), cur[k]));
        t = __dadd_rn(t, k > 1 ? __dmul_rn(be[k - 1], cur[k - 1]) : 0.0);
        t = __dsub_rn(t, __dmul_rn(bi, prev[k]));
        t = __dadd_rn(t, copysign(__dmul_rn(__dmul_rn(a.eps, __dadd_rn(be[k], b)), 0.3), t));
        const double wv = __ddiv_rn(t, b);
        nw[k] = wv;
        mx = fmax(mx, fabs(wv));
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) s_max[tid >> 5] = mx;
    __syncthreads();
    __shared__ int s_do;
    if (tid == 0) {
        double m2 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m2 = fmax(m2, s_max[w]);
        nw[it] = a.psi;
        nw[it + 1] = 1.0;
        const int thr = (it > 1) && (m2 > sqrt(a.eps));
        const int doit = *a.force || thr;
        *a.gate = doit;
        *a.force = thr;
        if (doit) *a.count += 1;
        s_do = doit;
    }
    __syncthreads();
    if (s_do)
        for (int k = 1 + tid; k <= it; k += blockDim.x) nw[k] = a.psi;
}

// ---------------------------------------------------------------------------
// a15: eigenvectors back to the original row order: out[k][r] = yt[inv[r]][k]
// (the caller's K x n_local buffer, vector k contiguous).
struct UnpermArgs {
    const void *yt;            // [ceil(K/KB)][npad][KB]
    const int32_t *inv;
    int64_t nrows, npad;
    int K;
    const int *k_found;
    void *const *out_ptr;
    const int *out_dtype;
};

__global__ void __launch_bounds__(kNT) k_unperm(UnpermArgs a) {
    void *out = *a.out_ptr;
    if (!out) return;
    const int kf = *a.k_found, dt = *a.out_dtype;
    for (int64_t r = (int64_t)blockIdx.x * kNT + threadIdx.x; r < a.nrows; r += (int64_t)gridDim.x * kNT) {
        const size_t p = (size_t)__ldg(a.inv + r);
        for (int k0 = 0; k0 < kf; k0 += kRitzKB) {
            const size_t src = ((size_t)(k0 / kRitzKB) * a.npad + p) * kRitzKB;
            if (dt == 0) {
                double g[kRitzKB];
#pragma unroll
                for (int q = 0; q < kRitzKB; q += 2) {
                    const double2 t = ld_stream(reinterpret_cast<const double2 *>(reinterpret_cast<const double *>(a.yt) + src + q));
                    g[q] = t.x;
                    g[q + 1] = t.y;
                }
#pragma unroll
                for (int q = 0; q < kRitzKB; ++q)
                    if (k0 + q < kf) __stcs(reinterpret_cast<double *>(out) + (size_t)(k0 + q) * a.nrows + r, g[q]);
            } else {
                float g[kRitzKB];
#pragma unroll
                for (int q = 0; q < kRitzKB; q += 4) {
                    const float4 t = ld_stream(reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(a.yt) + src + q));
                    g[q] = t.x; g[q + 1] = t.y; g[q + 2] = t.z; g[q + 3] = t.w;
                }
#pragma unroll
                for (int q = 0; q < kRitzKB; ++q)
                    if (k0 + q < kf) __stcs(reinterpret_cast<float *>(out) + (size_t)(k0 + q) * a.nrows + r, g[q]);
            }
        }
    }
}

}  // namespace topk
