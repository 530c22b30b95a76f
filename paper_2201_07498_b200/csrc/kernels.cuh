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
#include "device_common.cuh"
#include "host_prep.h"

namespace topk {

constexpr int kNT = 256;  // threads per block for the streaming kernels
constexpr int kRitzKB = 8;  // Ritz outputs per thread
constexpr int kStepJB = 8;  // basis columns per multi-dot pass of k_step

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
    double tau;
};

struct Exch {            // cross-part exchange buffers, slot g written by part g
    double *alpha_part;  // [G]
    double *hpart;       // [G][m+1]
    double *norm_part;   // [G]
    double *ritz_part;   // [G][K]
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
    __shared__ CT red[kNT / 32];
    __shared__ int sflag;
    constexpr int VW = Vw<ST>::N;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.st.done = 0;
        *a.st.m_found = 0;
        *a.st.tscale = 0.0;
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
        double tot = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, reinterpret_cast<double *>(red));
        if (threadIdx.x == 0) {
            a.ex.norm_part[a.g] = tot;
            *a.counter = 0;
        }
    }
}

// ---------------------------------------------------------------------------
// a7: SpMV + alpha partial (Alg.1 l.9-10), warp-per-tile segmented reduction.
// A warp owns a tile of whole non-empty rows (<= kTileNnz nonzeros) and walks
// it in rounds of 256 nonzeros: lane l holds 8 consecutive nonzeros (two
// 16-byte col loads, vector value loads, all L1::no_allocate streaming; the
// next round's columns and row-end bits are prefetched while the current round
// gathers). x is gathered through L1: hot columns (bit 31, the hub-first
// prefix of every slot) evict-last, the rest no_allocate. Products in the
// compute dtype; a lane-serial + warp-wide segmented scan over the row-end
// bitmask gives the row sums. Non-empty rows occupy positions [0, n_nonempty)
// in order, so the j-th row end of a tile is row end_begin + j. Rows longer
// than kTileNnz are chunked; the last-arriving chunk warp sums the chunk
// partials in chunk order. Epilogue: y_r = s_i * sum (deferred normalisation),
// stored once rounded, and the alpha partial sum_r y_r * v_i[r].
// Deterministic: fixed shuffle trees and fixed orders everywhere.
struct SpmvArgs {
    const int32_t *col;
    const void *val;
    const uint32_t *endbits;
    const Tile *tiles;
    int ntiles;
    const LongRow *longrows;
    double *long_parts;   // [ntiles]
    unsigned *long_cnt;   // [nlong]
    double *alpha_long;   // [nlong]
    int nlong;
    const void *x;        // gather source: V column it-1 (G = 1) or the replica
    const void *ui;       // local u_it (V column it-1)
    void *y;              // v_tmp (Q2), storage dtype
    double *y_dbg;        // optional fp64 unscaled row sums (debug export)
    double *slots;        // [grid]
    unsigned *counter;
    LzState st;
    Exch ex;
    int G, g;
};

// 8 consecutive matrix values (32-byte aligned group) converted to CT
template <typename VT, typename CT> struct Val8;
template <typename CT> struct Val8<float, CT> {
    static __device__ __forceinline__ void load(const float *p, CT (&o)[8]) {
        const float4 a = ld_stream(reinterpret_cast<const float4 *>(p));
        const float4 b = ld_stream(reinterpret_cast<const float4 *>(p) + 1);
        o[0] = (CT)a.x; o[1] = (CT)a.y; o[2] = (CT)a.z; o[3] = (CT)a.w;
        o[4] = (CT)b.x; o[5] = (CT)b.y; o[6] = (CT)b.z; o[7] = (CT)b.w;
    }
};
template <typename CT> struct Val8<double, CT> {
    static __device__ __forceinline__ void load(const double *p, CT (&o)[8]) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double2 a = ld_stream(reinterpret_cast<const double2 *>(p) + q);
            o[2 * q] = (CT)a.x;
            o[2 * q + 1] = (CT)a.y;
        }
    }
};
template <typename CT> struct Val8<bf16, CT> {
    static __device__ __forceinline__ void load(const bf16 *p, CT (&o)[8]) {
        const int4 v = ld_stream(reinterpret_cast<const int4 *>(p));
        const bf16 *e = reinterpret_cast<const bf16 *>(&v);
#pragma unroll
        for (int q = 0; q < 8; ++q) o[q] = cvt<CT>(e[q]);
    }
};

// x[c] for a remapped column entry: bit 31 set = hot column (kept in L1).
template <typename ST, typename CT>
__device__ __forceinline__ CT gather_x(const ST *__restrict__ x, int c) {
    if (c < 0) return cvt<CT>(ld_keep<ST>(x + (c & 0x7FFFFFFF)));
    return cvt<CT>(ld_noalloc<ST>(x + c));
}

template <typename VT, typename ST, typename CT>
__global__ void __launch_bounds__(kNT, 4) k_spmv(SpmvArgs a, int it) {
    constexpr int EPL = 8, RND = 32 * EPL;  // nonzeros per lane / per warp round
    __shared__ CT red[kNT / 32];
    __shared__ double redd[kNT / 32];
    __shared__ int sflag;

    double sd;
    if (!lz_prologue(it, a.st, a.ex, a.G, sd)) return;
    const CT s = (CT)sd;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int gwarp = (int)((blockIdx.x * kNT + threadIdx.x) >> 5);
    const int nwarps = (int)(gridDim.x * (kNT / 32));
    const VT *__restrict__ val = reinterpret_cast<const VT *>(a.val);
    const ST *__restrict__ x = reinterpret_cast<const ST *>(a.x);
    const ST *__restrict__ ui = reinterpret_cast<const ST *>(a.ui);
    ST *__restrict__ y = reinterpret_cast<ST *>(a.y);
    CT alpha_acc = CT(0);

    for (int t = gwarp; t < a.ntiles; t += nwarps) {
        const int4 T = __ldg(reinterpret_cast<const int4 *>(a.tiles) + t);
        const int zb = T.x, zend = T.x + T.y;
        const int z8 = zb & ~7;
        if (T.w < 0) {
            CT carry = CT(0);
            int jrow = T.z;
            // prefetch of round 0: columns + row-end bits
            int k0 = z8 + EPL * lane;
            int4 ca = make_int4(0, 0, 0, 0), cb = ca;
            unsigned wb = 0u;
            if (k0 < zend) {
                ca = ld_stream(reinterpret_cast<const int4 *>(a.col + k0));
                cb = ld_stream(reinterpret_cast<const int4 *>(a.col + k0) + 1);
                wb = __ldg(a.endbits + (k0 >> 5));
            }
            for (int base = z8; base < zend; base += RND) {
                const int cc[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
                const int kc = k0;
                const unsigned wcur = wb;
                k0 += RND;
                if (k0 < zend) {  // next round's columns in flight during this round's gathers
                    ca = ld_stream(reinterpret_cast<const int4 *>(a.col + k0));
                    cb = ld_stream(reinterpret_cast<const int4 *>(a.col + k0) + 1);
                    wb = __ldg(a.endbits + (k0 >> 5));
                }
                // valid-element mask of this lane's 8 slots: [zb, zend) intersect [kc, kc + 8)
                const int lo = max(zb - kc, 0), hi = min(zend - kc, EPL);
                const unsigned valid = (hi > lo) ? (((1u << hi) - 1u) & ~((1u << lo) - 1u)) : 0u;
                CT p[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) p[e] = CT(0);
                if (valid) {
                    CT v8[8];
                    Val8<VT, CT>::load(val + kc, v8);
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if ((valid >> e) & 1u) p[e] = v8[e] * gather_x<ST, CT>(x, cc[e]);
                }
                const unsigned fb = (wcur >> (kc & 31)) & valid & 0xFFu;
                // lane-serial segment sums
                CT part[8], run = CT(0), head = CT(0);
                bool seen = false;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    run += p[e];
                    part[e] = run;
                    if ((fb >> e) & 1u) {
                        if (!seen) { head = run; seen = true; }
                        run = CT(0);
                    }
                }
                // inclusive segmented scan of the open tails across lanes
                CT v = (lane == 0 && !seen) ? carry + run : run;
                int f = seen;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const CT vu = __shfl_up_sync(0xffffffffu, v, o);
                    const int fu = __shfl_up_sync(0xffffffffu, f, o);
                    if (lane >= o) {
                        if (!f) v = vu + v;
                        f |= fu;
                    }
                }
                CT cin = __shfl_up_sync(0xffffffffu, v, 1);
                if (lane == 0) cin = carry;
                carry = __shfl_sync(0xffffffffu, v, 31);
                // rank of this lane's row ends within the tile (ne <= 8)
                const unsigned ne = __popc(fb);
                const unsigned b0 = __ballot_sync(0xffffffffu, ne & 1u);
                const unsigned b1 = __ballot_sync(0xffffffffu, ne & 2u);
                const unsigned b2 = __ballot_sync(0xffffffffu, ne & 4u);
                const unsigned b3 = __ballot_sync(0xffffffffu, ne & 8u);
                int row = jrow + __popc(b0 & lt_mask) + 2 * __popc(b1 & lt_mask) + 4 * __popc(b2 & lt_mask) +
                          8 * __popc(b3 & lt_mask);
                jrow += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2) + 8 * __popc(b3);
                if (fb) {
                    bool first = true;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        if ((fb >> e) & 1u) {
                            const CT tot = first ? cin + head : part[e];
                            first = false;
                            const CT yv = s * tot;
                            y[row] = rnd_ct<ST, CT>(yv);
                            alpha_acc += yv * (s * cvt<CT>(ld_noalloc<ST>(ui + row)));
                            if (a.y_dbg) a.y_dbg[row] = (double)tot;
                            ++row;
                        }
                    }
                }
            }
        } else {
            // chunk of a long row: warp partial, last-arriving chunk finishes the row
            CT part = CT(0);
            for (int base = z8; base < zend; base += RND) {
                const int kc = base + EPL * lane;
                const int lo = max(zb - kc, 0), hi = min(zend - kc, EPL);
                if (hi > lo) {
                    const unsigned valid = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
                    const int4 ca = ld_stream(reinterpret_cast<const int4 *>(a.col + kc));
                    const int4 cb = ld_stream(reinterpret_cast<const int4 *>(a.col + kc) + 1);
                    const int cc[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
                    CT v8[8];
                    Val8<VT, CT>::load(val + kc, v8);
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if ((valid >> e) & 1u) part += v8[e] * gather_x<ST, CT>(x, cc[e]);
                }
            }
            part = warp_sum(part);
            if (lane == 0) {
                const LongRow L = a.longrows[T.w];
                a.long_parts[t] = (double)part;
                __threadfence();
                const unsigned prev = atomicAdd(a.long_cnt + T.w, 1u);
                if (prev == (unsigned)L.nchunks - 1) {
                    __threadfence();
                    CT sum = CT(0);
                    for (int q = 0; q < L.nchunks; ++q) sum += (CT)__ldcg(a.long_parts + L.first_tile + q);
                    const CT yv = s * sum;
                    y[L.row] = rnd_ct<ST, CT>(yv);
                    a.alpha_long[T.w] = (double)(yv * (s * cvt<CT>(ui[L.row])));
                    if (a.y_dbg) a.y_dbg[L.row] = (double)sum;
                    a.long_cnt[T.w] = 0u;
                }
            }
        }
    }
    const CT tot = block_sum<CT, kNT>(alpha_acc, red);
    if (threadIdx.x == 0) a.slots[blockIdx.x] = (double)tot;
    if (arrive_last(a.counter, &sflag)) {
        const double s1 = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, redd);
        const double s2 = block_sum_array<double, kNT>(a.alpha_long, a.nlong, 1, redd);
        if (threadIdx.x == 0) {
            a.ex.alpha_part[a.g] = s1 + s2;
            *a.counter = 0u;
        }
    }
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
};

template <typename ST, typename CT, int JB>
__global__ void __launch_bounds__(kNT, 4) k_step(StepArgs a, int it) {
    constexpr int VW = Vw<ST>::N;
    __shared__ CT part[kNT / 32][JB];
    __shared__ CT red[kNT / 32];
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
        c2 = (it > 1) ? (CT)(bi * a.st.scale[it - 2]) : CT(0);    // beta_i * s_{i-1}
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
            const double tot = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, reinterpret_cast<double *>(red));
            if (tid == 0) { a.ex.norm_part[a.g] = tot; *a.counter = 0u; }
        }
        return;
    }

    // Multi-dot h_j = u_j . w: the block's threads form NG column groups of LPG
    // lanes; group g takes columns j0 + g*JB .. +JB-1 for the SAME rows, so one
    // pass over the rows streams every basis column from DRAM once (y, u_i,
    // u_{i-1}, w are re-read by the other groups from L1/L2) while each thread
    // keeps only JB accumulators. Passes over further column blocks (it > NG*JB)
    // read the stored w.
    constexpr int NG = 4, LPG = kNT / NG;
    const int grp = tid / LPG, gl = tid - grp * LPG;
    for (int jb0 = 0; jb0 < it; jb0 += NG * JB) {
        const int j0 = jb0 + grp * JB;
        CT acc[JB];
#pragma unroll
        for (int q = 0; q < JB; ++q) acc[q] = CT(0);
        for (int64_t v = (int64_t)blockIdx.x * LPG + gl; v < nvec; v += (int64_t)gridDim.x * LPG) {
            CT w[VW];
            if (a.mode == 2) {
                vload<ST, CT>(src2 + v * VW, w);
            } else if (jb0 == 0) {
                CT yy[VW], u1[VW], u0[VW];
                vload<ST, CT>(yv + v * VW, yy);
                vload<ST, CT>(ucur + v * VW, u1);
                if (it > 1) vload<ST, CT>(uprev + v * VW, u0);
#pragma unroll
                for (int q = 0; q < VW; ++q) w[q] = yy[q] - c1 * u1[q] - (it > 1 ? c2 * u0[q] : CT(0));
                // w rounded once; every group dots with the rounded (stored) value
                if (grp == 0) vstore_back<ST, CT>(wv + v * VW, w);
                else round_back<ST, CT>(w);
            } else {
                vload<ST, CT>(wv + v * VW, w);
            }
#pragma unroll
            for (int q = 0; q < JB; ++q) {
                const int j = j0 + q;
                if (j < it) {
                    CT u[VW];
                    vload<ST, CT>(V + (size_t)j * a.npad + v * VW, u);
                    CT d = CT(0);
#pragma unroll
                    for (int e = 0; e < VW; ++e) d += u[e] * w[e];
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
        if (tid < NG * JB && jb0 + tid < it) {  // column jb0 + tid = group tid / JB, slot tid % JB
            constexpr int WPG = LPG / 32;
            const int g2 = tid / JB, q = tid - g2 * JB;
            CT r = CT(0);
#pragma unroll
            for (int w8 = 0; w8 < WPG; ++w8) r += part[g2 * WPG + w8][q];
            a.slots[(size_t)blockIdx.x * a.ld + jb0 + tid] = (double)r;
        }
        __syncthreads();
    }
    if (arrive_last(a.counter, &sflag)) {
        // warp w sums column j = w, w+8, ...: lanes stride the block slots
        for (int j = wid; j < it; j += kNT / 32) {
            double r = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) r += __ldcg(a.slots + (size_t)b * a.ld + j);
            r = warp_sum(r);
            if (lane == 0) a.ex.hpart[(size_t)a.g * a.ld + j] = r;
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
};

template <typename ST, typename CT>
__global__ void __launch_bounds__(kNT) k_correct(CorrArgs a, int it) {
    constexpr int VW = Vw<ST>::N;
    extern __shared__ double dsm[];  // coef[it]
    __shared__ CT red[kNT / 32];
    __shared__ int sflag;
    if (*(volatile int *)a.st.done) return;
    const int tid = threadIdx.x;
    CT *coef = reinterpret_cast<CT *>(dsm);
    for (int j = tid; j < it; j += kNT) {
        double h = 0.0;
        for (int q = 0; q < a.G; ++q) h += __ldcg(a.ex.hpart + (size_t)q * a.ld + j);
        const double sj = a.st.scale[j];
        coef[j] = (CT)(h * sj * sj);
    }
    __syncthreads();
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
        const double tot = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, reinterpret_cast<double *>(red));
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
};

__device__ __forceinline__ int rr_player(int pos, int round, int M) {
    if (pos == 0) return 0;
    int x = pos - 1 + round;
    if (x >= M - 1) x -= M - 1;
    return 1 + x;
}

template <bool kSmem>
__global__ void k_jacobi(JacArgs a) {
    extern __shared__ double jsm[];
    __shared__ int s_rot;
    __shared__ double s_fro;
    const int tid = threadIdx.x, nt = blockDim.x;
    const LzState &st = a.st;
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
    for (int i = tid; i < M * LD; i += nt) {
        const int r = i >> LS, c = i & (LD - 1);
        double t = 0.0;
        if (r < mm && c < mm) {
            if (r == c) t = st.alpha[r];
            else if (r - c == 1 || c - r == 1) t = st.beta[r > c ? r : c];
        }
        T[i] = t;
        S[i] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (tid == 0) {
        double f = 0.0;  // ||T||_F in the oracle's summation order (row-major)
        for (int r = 0; r < mm; ++r)
            for (int c = 0; c < mm; ++c) f += T[(r << LS) + c] * T[(r << LS) + c];
        s_fro = sqrt(f);
    }
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
                    const double apq = T[(p << LS) + q], app = T[(p << LS) + p], aqq = T[(q << LS) + q];
                    const double a2 = apq * apq;
                    if (!(a2 <= eps * eps * fabs(app * aqq) || a2 <= fro2)) {
                        const double d = aqq - app;
                        const bool zpos = (d == 0.0) || ((d > 0.0) == (apq > 0.0));
                        const double x = d * d + 4.0 * a2;
                        const double D = fabs(d) + x * rsqrt(x);
                        const double ih = rsqrt(D * D + 4.0 * a2);
                        c = D * ih;
                        sn = (zpos ? 2.0 : -2.0) * fabs(apq) * ih;
                        doit = 1;
                        s_rot = 1;
                    }
                }
                cs[2 * k] = c;
                cs[2 * k + 1] = sn;
                rot[k] = doit;
            }
            __syncthreads();
            // phase B1: T <- J^T T J as 2x2 blocks (rows of pair k, columns of pair l)
            for (int i = tid; i < (half << HS); i += nt) {
                const int k = i >> HS, l = i & (HD - 1);
                if (l >= half || !(rot[k] | rot[l])) continue;
                const int pk = pq[2 * k], qk = pq[2 * k + 1], pl = pq[2 * l], ql = pq[2 * l + 1];
                const double ck = cs[2 * k], sk = cs[2 * k + 1], cl = cs[2 * l], sl = cs[2 * l + 1];
                double *r0 = T + (pk << LS), *r1 = T + (qk << LS);
                const double b00 = r0[pl], b01 = r0[ql], b10 = r1[pl], b11 = r1[ql];
                const double e00 = cl * b00 - sl * b01, e01 = sl * b00 + cl * b01;  // columns (T J)
                const double e10 = cl * b10 - sl * b11, e11 = sl * b10 + cl * b11;
                r0[pl] = ck * e00 - sk * e10;                                      // rows (J^T .)
                r1[pl] = sk * e00 + ck * e10;
                if (k == l && rot[k]) {
                    r0[ql] = 0.0;
                    r1[pl] = 0.0;
                } else {
                    r0[ql] = ck * e01 - sk * e11;
                }
                r1[ql] = sk * e01 + ck * e11;
            }
            // phase B2: S <- S J (columns p, q), row r
            for (int i = tid; i < (half << LS); i += nt) {
                const int k = i >> LS, r = i & (LD - 1);
                if (r >= mm || !rot[k]) continue;
                const int p = pq[2 * k], q = pq[2 * k + 1];
                const double c = cs[2 * k], sn = cs[2 * k + 1];
                double *Sr = S + (r << LS);
                const double sp = Sr[p], sq = Sr[q];
                Sr[p] = c * sp - sn * sq;
                Sr[q] = sn * sp + c * sq;
            }
            __syncthreads();
        }
        ++sweeps;
        conv = !s_rot;
        __syncthreads();
    }
    // selection + sign + outputs
    const int K = a.K;
    const int kf = K < mm ? K : mm;
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
        }
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

// ---------------------------------------------------------------------------
// a14: Ritz projection y_k = sum_j S[j,k] v_j ("the eigenvectors of
// M are given by 𝒱V"), fp64 accumulation, then y_k / ||y_k|| (reading Q12).
// Two streaming passes over the stored basis; no fp64 Y is materialised:
//   pass 0: recompute y_k row by row, per-block partials of ||y_k||^2 ->
//           ex.ritz_part[g][k] (last-arriving block per output group, fixed order)
//   pass 1: recompute y_k, scale by 1/||y_k|| (norms summed over parts in rank
//           order) and store once, in the output dtype, to the caller's buffer
//           in ORIGINAL row order (position p -> row perm[p]; hub-first order
//           keeps all non-hot rows ascending, so the stores stay coalesced).
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
    void *const *out_ptr;     // device param: output base (K vectors of nrows)
    const int *out_dtype;     // device param: 0 f64, 1 f32
    const int32_t *perm;      // position -> part-local original row (output order)
};

template <typename ST, typename CT, int KB>
__global__ void __launch_bounds__(kNT, 2) k_ritz(RitzArgs a, int pass) {
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
        for (int j = 0; j < mm; ++j) {
            CT u[VW];
            vload_cs<ST, CT>(V + (size_t)j * a.npad + v * VW, u);
            const CT *cj = coef + j * KB;
#pragma unroll
            for (int q = 0; q < KB; ++q) {
                const CT c = cj[q];
#pragma unroll
                for (int e = 0; e < VW; ++e) acc[e][q] += c * u[e];
            }
        }
        if (pass == 0) {
#pragma unroll
            for (int q = 0; q < KB; ++q)
#pragma unroll
                for (int e = 0; e < VW; ++e) nrm[q] += acc[e][q] * acc[e][q];
        } else {
            int32_t orow[VW];
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                const int64_t r = v * VW + e;
                orow[e] = (r < a.nrows) ? __ldg(a.perm + r) : 0;
            }
#pragma unroll
            for (int q = 0; q < KB; ++q) {
                if (k0 + q >= kf) break;
                const double iv = inv[q];
                const size_t base = (size_t)(k0 + q) * a.nrows;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const int64_t r = v * VW + e;
                    if (r < a.nrows) {
                        const size_t o = base + (size_t)orow[e];
                        const double yv = (double)acc[e][q] * iv;
                        if (dt == 0) __stcs(reinterpret_cast<double *>(out) + o, yv);
                        else __stcs(reinterpret_cast<float *>(out) + o, (float)yv);
                    }
                }
            }
        }
    }
    if (pass == 1) return;
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

}  // namespace topk
