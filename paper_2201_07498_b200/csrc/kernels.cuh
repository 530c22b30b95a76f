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
    const double *v1;      // device, n_g doubles (if *use_v1)
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
                if (use_v1) x = a.v1[r];
                else {
                    uint64_t h = mix64(hs ^ (uint64_t)(a.row0 + r));
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
// a7: SpMV + alpha partial (Alg.1 l.9-10). nnz-tiled: a packed tile holds whole
// rows with <= kTileNnz nonzeros; each of 256 threads owns 8 consecutive
// nonzeros; products go to shared memory, a block-wide segmented scan sums rows
// (balanced regardless of the power-law row lengths); rows longer than a tile
// are split into chunks finished by the last-arriving chunk block.
struct SpmvArgs {
    const int32_t *rowptr;
    const int32_t *col;
    const void *val;
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

__device__ __forceinline__ int padi(int e) { return e + (e >> 3); }

template <typename VT, typename ST, typename CT>
__global__ void __launch_bounds__(kNT) k_spmv(SpmvArgs a, int it) {
    constexpr int IPT = kTileNnz / kNT;  // 8
    __shared__ CT prod[kTileNnz + kTileNnz / 8];
    __shared__ __align__(16) uint8_t flags[kTileNnz];
    __shared__ int32_t rp[kTileRows + 1];
    __shared__ CT wv[kNT / 32];
    __shared__ int wf[kNT / 32];
    __shared__ CT red[kNT / 32];
    __shared__ int sflag;

    double sd;
    if (!lz_prologue(it, a.st, a.ex, a.G, sd)) return;
    const CT s = (CT)sd;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const VT *__restrict__ val = reinterpret_cast<const VT *>(a.val);
    const ST *__restrict__ x = reinterpret_cast<const ST *>(a.x);
    const ST *__restrict__ ui = reinterpret_cast<const ST *>(a.ui);
    ST *__restrict__ y = reinterpret_cast<ST *>(a.y);
    CT alpha_acc = CT(0);

    for (int t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        const Tile T = a.tiles[t];
        if (T.long_id < 0) {
            const int rb = T.row_begin, nr = T.row_end - T.row_begin, nzb = T.nz_begin;
            const int cnt = __ldg(a.rowptr + T.row_end) - nzb;
            // issue the streaming loads of this tile's nonzeros first (MLP)
            int32_t c[IPT];
            VT v[IPT];
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                const int k = j * kNT + tid;
                if (k < cnt) {
                    c[j] = __ldcs(a.col + nzb + k);
                    v[j] = __ldcs(val + nzb + k);
                }
            }
            for (int q = tid; q <= nr; q += kNT) rp[q] = __ldg(a.rowptr + rb + q) - nzb;
            *reinterpret_cast<uint2 *>(&flags[tid * IPT]) = make_uint2(0u, 0u);
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                const int k = j * kNT + tid;
                if (k < cnt) prod[padi(k)] = cvt<CT>(v[j]) * cvt<CT>(__ldg(x + c[j]));
            }
            __syncthreads();
            for (int q = tid; q < nr; q += kNT)
                if (rp[q] < rp[q + 1]) flags[rp[q]] = 1;
            __syncthreads();
            // per-thread segmented inclusive scan over its 8 elements
            const int e0 = tid * IPT;
            CT run = CT(0);
            int any = 0, first = IPT;
            const uint2 fl = *reinterpret_cast<const uint2 *>(&flags[e0]);
            const uint8_t *fb = reinterpret_cast<const uint8_t *>(&fl);
#pragma unroll
            for (int q = 0; q < IPT; ++q) {
                const int e = e0 + q;
                if (e < cnt) {
                    const CT pv = prod[padi(e)];
                    if (fb[q]) {
                        run = pv;
                        if (!any) { any = 1; first = q; }
                    } else {
                        run += pv;
                    }
                    prod[padi(e)] = run;
                }
            }
            // block-wide exclusive segmented scan of (any, run)
            int f = any;
            CT sv = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int fu = __shfl_up_sync(0xffffffffu, f, o);
                const CT vu = __shfl_up_sync(0xffffffffu, sv, o);
                if (lane >= o) {
                    if (!f) sv = vu + sv;
                    f |= fu;
                }
            }
            if (lane == 31) { wf[wid] = f; wv[wid] = sv; }
            int fe = __shfl_up_sync(0xffffffffu, f, 1);
            CT ve = __shfl_up_sync(0xffffffffu, sv, 1);
            if (lane == 0) { fe = 0; ve = CT(0); }
            __syncthreads();
            CT pv = CT(0);
            int pf = 0;
            for (int w = 0; w < wid; ++w) {  // prefix over previous warps, fixed order
                if (wf[w]) { pv = wv[w]; pf = 1; } else { pv = pv + wv[w]; }
            }
            const CT carry = fe ? ve : pv + ve;
            (void)pf;
            if (tid > 0) {
#pragma unroll
                for (int q = 0; q < IPT; ++q) {
                    const int e = e0 + q;
                    if (q < first && e < cnt) prod[padi(e)] = carry + prod[padi(e)];
                }
            }
            __syncthreads();
            for (int q = tid; q < nr; q += kNT) {
                const int e = rp[q + 1] - 1;
                const CT sum = (rp[q] <= e) ? prod[padi(e)] : CT(0);
                const CT yv = s * sum;
                y[rb + q] = rnd_ct<ST, CT>(yv);
                alpha_acc += yv * (s * cvt<CT>(ui[rb + q]));
                if (a.y_dbg) a.y_dbg[rb + q] = (double)sum;
            }
            __syncthreads();
        } else {
            const LongRow L = a.longrows[T.long_id];
            const int r = T.row_begin, nzb = T.nz_begin;
            const int cnt = min(kTileNnz, __ldg(a.rowptr + r + 1) - nzb);
            CT part = CT(0);
#pragma unroll
            for (int j = 0; j < IPT; ++j) {
                const int k = j * kNT + tid;
                if (k < cnt) part += cvt<CT>(__ldcs(val + nzb + k)) * cvt<CT>(__ldg(x + __ldcs(a.col + nzb + k)));
            }
            part = block_sum<CT, kNT>(part, red);
            if (tid == 0) {
                a.long_parts[t] = (double)part;
                __threadfence();
                const unsigned prev = atomicAdd(a.long_cnt + T.long_id, 1u);
                if (prev == (unsigned)L.nchunks - 1) {
                    __threadfence();
                    CT sum = CT(0);
                    for (int q = 0; q < L.nchunks; ++q) sum += (CT)__ldcg(a.long_parts + L.first_tile + q);
                    const CT yv = s * sum;
                    y[r] = rnd_ct<ST, CT>(yv);
                    a.alpha_long[T.long_id] = (double)(yv * (s * cvt<CT>(ui[r])));
                    if (a.y_dbg) a.y_dbg[r] = (double)sum;
                    a.long_cnt[T.long_id] = 0u;
                }
            }
        }
    }
    const CT tot = block_sum<CT, kNT>(alpha_acc, red);
    if (tid == 0) a.slots[blockIdx.x] = (double)tot;
    if (arrive_last(a.counter, &sflag)) {
        double* rd = reinterpret_cast<double *>(prod);
        const double s1 = block_sum_array<double, kNT>(a.slots, gridDim.x, 1, rd);
        const double s2 = block_sum_array<double, kNT>(a.alpha_long, a.nlong, 1, rd);
        if (tid == 0) {
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
__global__ void __launch_bounds__(kNT) k_step(StepArgs a, int it) {
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

    for (int j0 = 0; j0 < it; j0 += JB) {
        CT acc[JB];
#pragma unroll
        for (int q = 0; q < JB; ++q) acc[q] = CT(0);
        for (int64_t v = (int64_t)blockIdx.x * kNT + tid; v < nvec; v += (int64_t)gridDim.x * kNT) {
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
        if (tid < JB && j0 + tid < it) {
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
    for (int64_t v = (int64_t)blockIdx.x * kNT + tid; v < nvec; v += (int64_t)gridDim.x * kNT) {
        CT acc[VW];
        vload<ST, CT>(src + v * VW, acc);
        for (int j = 0; j < it; ++j) {
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
// a12-a13: Jacobi on T in one block, parallel (round-robin
// tournament) ordering of the same rotations as the oracle's cyclic ordering;
// same negligibility rule (|t_pq| <= eps sqrt|t_pp t_qq| or <= eps^2 ||T||_F);
// then top-K by (-|theta|, -theta) and the sign convention s_1k > 0.
struct JacArgs {
    LzState st;
    Exch ex;
    int G, m, K, max_sweeps;
    double *work;  // global fallback workspace (2 * M * M doubles) or nullptr
    int use_smem;
};

__device__ __forceinline__ int rr_player(int pos, int round, int M) {
    return pos == 0 ? 0 : 1 + (pos - 1 + round) % (M - 1);
}

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
    double *T = a.use_smem ? jsm : a.work;
    double *S = T + (size_t)M * M;
    int *rot = reinterpret_cast<int *>(S + (size_t)M * M);           // [M/2]
    double *cs = reinterpret_cast<double *>(rot + ((M / 2 + 1) & ~1));  // [M/2][2]
    for (int i = tid; i < M * M; i += nt) {
        const int r = i / M, c = i % M;
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
        double f = 0.0;
        for (int i = 0; i < M * M; ++i) f += T[i] * T[i];
        s_fro = sqrt(f);
    }
    __syncthreads();
    const double eps = 2.220446049250313e-16;
    const double fro = s_fro;
    int sweeps = 0, conv = (M < 2) ? 1 : 0;
    const int half = M / 2;
    while (!conv && sweeps < a.max_sweeps) {
        if (tid == 0) s_rot = 0;
        __syncthreads();
        for (int round = 0; round < M - 1; ++round) {
            for (int k = tid; k < half; k += nt) {
                int p = rr_player(k, round, M), q = rr_player(M - 1 - k, round, M);
                if (p > q) { int t = p; p = q; q = t; }
                int doit = 0;
                if (q < mm) {
                    const double apq = T[p * M + q], app = T[p * M + p], aqq = T[q * M + q];
                    if (fabs(apq) <= eps * sqrt(fabs(app * aqq)) || fabs(apq) <= eps * eps * fro) {
                        T[p * M + q] = 0.0;
                        T[q * M + p] = 0.0;
                    } else {
                        const double zeta = (aqq - app) / (2.0 * apq);
                        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                        const double c = 1.0 / sqrt(1.0 + t * t);
                        cs[2 * k] = c;
                        cs[2 * k + 1] = t * c;
                        doit = 1;
                        s_rot = 1;
                    }
                }
                rot[k] = doit;
            }
            __syncthreads();
            for (int i = tid; i < half * M; i += nt) {  // T <- T J, S <- S J (columns p, q)
                const int k = i / M, r = i % M;
                if (!rot[k]) continue;
                int p = rr_player(k, round, M), q = rr_player(M - 1 - k, round, M);
                if (p > q) { int t = p; p = q; q = t; }
                const double c = cs[2 * k], s = cs[2 * k + 1];
                const double tp = T[r * M + p], tq = T[r * M + q];
                T[r * M + p] = c * tp - s * tq;
                T[r * M + q] = s * tp + c * tq;
                const double sp = S[r * M + p], sq = S[r * M + q];
                S[r * M + p] = c * sp - s * sq;
                S[r * M + q] = s * sp + c * sq;
            }
            __syncthreads();
            for (int i = tid; i < half * M; i += nt) {  // T <- J^T T (rows p, q)
                const int k = i / M, col = i % M;
                if (!rot[k]) continue;
                int p = rr_player(k, round, M), q = rr_player(M - 1 - k, round, M);
                if (p > q) { int t = p; p = q; q = t; }
                const double c = cs[2 * k], s = cs[2 * k + 1];
                const double tp = T[p * M + col], tq = T[q * M + col];
                T[p * M + col] = c * tp - s * tq;
                T[q * M + col] = s * tp + c * tq;
            }
            __syncthreads();
            for (int k = tid; k < half; k += nt) {
                if (!rot[k]) continue;
                int p = rr_player(k, round, M), q = rr_player(M - 1 - k, round, M);
                T[p * M + q] = 0.0;
                T[q * M + p] = 0.0;
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
        const double tc = T[c * M + c];
        st.theta_all[c] = tc;
        int rank = 0;
        for (int d = 0; d < mm; ++d) {
            const double td = T[d * M + d];
            const bool before = (fabs(td) != fabs(tc)) ? (fabs(td) > fabs(tc))
                                : (td != tc) ? (td > tc) : (d < c);
            rank += before;
        }
        if (rank < kf) {
            double sg = 1.0;
            for (int j = 0; j < mm; ++j) {
                const double sj = S[j * M + c];
                if (sj != 0.0) { sg = sj > 0.0 ? 1.0 : -1.0; break; }
            }
            st.evals[rank] = tc;
            for (int j = 0; j < mm; ++j) st.coefS[(size_t)j * K + rank] = sg * S[j * M + c] * st.scale[j];
            st.resid[rank] = fabs(st.beta[mm] * S[(mm - 1) * M + c]);
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
// a14: Ritz projection Y = V S_K ("𝒱V") with fp64 accumulation,
// per-block squared-norm partials; k_ritz_norm scales to unit norm.
struct RitzArgs {
    const void *V;
    double *Y;        // [K][npad] unnormalised
    int64_t npad, nrows;
    int K;
    double *slots;    // [grid][K]
    unsigned *counter;
    LzState st;
    Exch ex;
    int g;
};

template <typename ST, typename CT, int KB>
__global__ void __launch_bounds__(kNT) k_ritz(RitzArgs a) {
    extern __shared__ double rsm[];  // coef[m' * K]
    __shared__ CT part[kNT / 32][KB];
    __shared__ int sflag;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int mm = *a.st.m_found, kf = *a.st.k_found, K = a.K;
    CT *coef = reinterpret_cast<CT *>(rsm);
    for (int i = tid; i < mm * K; i += kNT) coef[i] = (CT)a.st.coefS[i];
    __syncthreads();
    const ST *V = reinterpret_cast<const ST *>(a.V);
    for (int k0 = 0; k0 < kf; k0 += KB) {
        CT nrm[KB];
#pragma unroll
        for (int q = 0; q < KB; ++q) nrm[q] = CT(0);
        for (int64_t r = (int64_t)blockIdx.x * kNT + tid; r < a.nrows; r += (int64_t)gridDim.x * kNT) {
            CT acc[KB];
#pragma unroll
            for (int q = 0; q < KB; ++q) acc[q] = CT(0);
            for (int j = 0; j < mm; ++j) {
                const CT u = cvt<CT>(V[(size_t)j * a.npad + r]);
                const CT *cj = coef + (size_t)j * K + k0;
#pragma unroll
                for (int q = 0; q < KB; ++q)
                    if (k0 + q < kf) acc[q] += cj[q] * u;
            }
#pragma unroll
            for (int q = 0; q < KB; ++q)
                if (k0 + q < kf) {
                    a.Y[(size_t)(k0 + q) * a.npad + r] = (double)acc[q];
                    nrm[q] += acc[q] * acc[q];
                }
        }
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
            a.slots[(size_t)blockIdx.x * K + k0 + tid] = (double)rr;
        }
        __syncthreads();
    }
    if (arrive_last(a.counter, &sflag)) {
        for (int k = wid; k < kf; k += kNT / 32) {
            double rr = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) rr += __ldcg(a.slots + (size_t)b * K + k);
            rr = warp_sum(rr);
            if (lane == 0) a.ex.ritz_part[(size_t)a.g * K + k] = rr;
        }
        __syncthreads();
        if (tid == 0) *a.counter = 0u;
    }
}

struct RitzNormArgs {
    const double *Y;
    int64_t npad, nrows;
    int K, G;
    const int *k_found;
    const double *ritz_part;  // [G][K]
    void *const *out_ptr;     // device param: output base (K vectors of nrows)
    const int *out_dtype;     // device param: 0 f64, 1 f32
};

__global__ void __launch_bounds__(kNT) k_ritz_norm(RitzNormArgs a) {
    __shared__ double inv[256];
    const int kf = *a.k_found;
    void *out = *a.out_ptr;
    if (!out) return;
    for (int k = threadIdx.x; k < kf && k < 256; k += blockDim.x) {
        double s = 0.0;
        for (int q = 0; q < a.G; ++q) s += __ldcg(a.ritz_part + (size_t)q * a.K + k);
        inv[k] = 1.0 / sqrt(s);
    }
    __syncthreads();
    const int dt = *a.out_dtype;
    const int64_t total = (int64_t)kf * a.nrows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / a.nrows);
        const int64_t r = i - (int64_t)k * a.nrows;
        const double v = a.Y[(size_t)k * a.npad + r] * inv[k];
        if (dt == 0) reinterpret_cast<double *>(out)[i] = v;
        else reinterpret_cast<float *>(out)[i] = (float)v;
    }
}

}  // namespace topk
