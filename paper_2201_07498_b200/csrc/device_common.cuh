// device_common.cuh — storage/compute dtype plumbing, deterministic reductions,
// last-block finalisation. sm_100a only.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace topk {

// Device-side checks of a dev build variant (tools/build.py build_variant with
// TOPK_CHECKS; tools/check_run.sh): bounds of every gather / scatter index and the
// ticket counters of the last-block reductions. A failed check prints and traps.
// compute-sanitizer is not available on this GPU pool, so these replace it.
#ifdef TOPK_CHECKS
#define TOPK_DCHECK(cond, what)                                                              \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("TOPK_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__,    \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define TOPK_DCHECK(cond, what) do { } while (0)
#endif

using bf16 = __nv_bfloat16;

// ---- storage dtype traits: vector width for 16-byte loads -------------------
template <typename T> struct Vw;
template <> struct Vw<double> { static constexpr int N = 2; };
template <> struct Vw<float> { static constexpr int N = 4; };
template <> struct Vw<bf16> { static constexpr int N = 8; };

template <typename CT> __device__ __forceinline__ CT to_ct(double x) { return (CT)x; }
template <typename CT> __device__ __forceinline__ CT cvt(double x) { return (CT)x; }
template <typename CT> __device__ __forceinline__ CT cvt(float x) { return (CT)x; }
template <typename CT> __device__ __forceinline__ CT cvt(bf16 x) { return (CT)__bfloat162float(x); }

// round-to-nearest-even once on store (reading Q14)
template <typename ST> __device__ __forceinline__ ST rnd(double x);
template <> __device__ __forceinline__ double rnd<double>(double x) { return x; }
template <> __device__ __forceinline__ float rnd<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ bf16 rnd<bf16>(double x) { return __double2bfloat16(x); }
template <typename ST> __device__ __forceinline__ ST rndf(float x);
template <> __device__ __forceinline__ double rndf<double>(float x) { return (double)x; }
template <> __device__ __forceinline__ float rndf<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 rndf<bf16>(float x) { return __float2bfloat16_rn(x); }
template <typename ST, typename CT> __device__ __forceinline__ ST rnd_ct(CT x) {
    if constexpr (sizeof(CT) == 8) return rnd<ST>((double)x);
    else return rndf<ST>((float)x);
}

// 16-byte vector load/store of N = Vw<ST>::N storage elements, converted to CT.
template <typename ST, typename CT>
__device__ __forceinline__ void vload(const ST *__restrict__ p, CT (&o)[Vw<ST>::N]) {
    uint4 raw = __ldg(reinterpret_cast<const uint4 *>(p));
    const ST *e = reinterpret_cast<const ST *>(&raw);
#pragma unroll
    for (int q = 0; q < Vw<ST>::N; ++q) o[q] = cvt<CT>(e[q]);
}
// streaming (evict-first) variant for data read once per kernel
template <typename ST, typename CT>
__device__ __forceinline__ void vload_cs(const ST *__restrict__ p, CT (&o)[Vw<ST>::N]) {
    uint4 raw = __ldcs(reinterpret_cast<const uint4 *>(p));
    const ST *e = reinterpret_cast<const ST *>(&raw);
#pragma unroll
    for (int q = 0; q < Vw<ST>::N; ++q) o[q] = cvt<CT>(e[q]);
}
template <typename ST, typename CT>
__device__ __forceinline__ void vstore(ST *__restrict__ p, const CT (&v)[Vw<ST>::N]) {
    uint4 raw;
    ST *e = reinterpret_cast<ST *>(&raw);
#pragma unroll
    for (int q = 0; q < Vw<ST>::N; ++q) e[q] = rnd_ct<ST, CT>(v[q]);
    *reinterpret_cast<uint4 *>(p) = raw;
}
// store rounded and return the rounded values in CT (what was stored)
template <typename ST, typename CT>
__device__ __forceinline__ void vstore_back(ST *__restrict__ p, CT (&v)[Vw<ST>::N]) {
    uint4 raw;
    ST *e = reinterpret_cast<ST *>(&raw);
#pragma unroll
    for (int q = 0; q < Vw<ST>::N; ++q) {
        e[q] = rnd_ct<ST, CT>(v[q]);
        v[q] = cvt<CT>(e[q]);
    }
    *reinterpret_cast<uint4 *>(p) = raw;
}

// round to the storage dtype and back (the value vstore_back would store)
template <typename ST, typename CT>
__device__ __forceinline__ void round_back(CT (&v)[Vw<ST>::N]) {
#pragma unroll
    for (int q = 0; q < Vw<ST>::N; ++q) v[q] = cvt<CT>(rnd_ct<ST, CT>(v[q]));
}

// ---- L1 cache-policy loads (read-only path) ----------------------------------
// stream: data read exactly once per kernel (matrix col/val) must not displace
// the x values kept in L1 -> L1::no_allocate; the SpMV gathers x with plain
// (L1-allocating) __ldg, DESIGN.md section 7.
__device__ __forceinline__ int4 ld_stream(const int4 *p) {
    int4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float4 ld_stream(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ld_stream(const double2 *p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_stream(const uint2 *p) {
    uint2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
template <typename T> __device__ __forceinline__ T ld_noalloc(const T *p);
template <> __device__ __forceinline__ float ld_noalloc<float>(const float *p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
template <> __device__ __forceinline__ double ld_noalloc<double>(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
template <> __device__ __forceinline__ bf16 ld_noalloc<bf16>(const bf16 *p) {
    unsigned short v;
    asm volatile("ld.global.nc.L1::no_allocate.b16 %0, [%1];" : "=h"(v) : "l"(p));
    return __ushort_as_bfloat16(v);
}

// ---- TMA bulk copies + mbarrier (global -> shared, completion by tx bytes) ----
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MBAR_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- deterministic reductions (fixed shuffle tree + fixed warp order) --------
template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// Result valid in thread 0. `sm` needs NT/32 elements. Ends with a barrier.
template <typename T, int NT> __device__ __forceinline__ T block_sum(T v, T *sm) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sm[w] = v;
    __syncthreads();
    T r = T(0);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) r += sm[i];
    }
    __syncthreads();
    return r;
}

// Sum n values of a global array in fixed order using the whole block.
// Result valid in thread 0.
template <typename T, int NT>
__device__ __forceinline__ T block_sum_array(const T *a, int n, int stride, T *sm) {
    T s = T(0);
    for (int i = threadIdx.x; i < n; i += NT) s += __ldcg(a + (size_t)i * stride);
    return block_sum<T, NT>(s, sm);
}

// Classic threadfence "last block" pattern: every block publishes its partial,
// then the block that arrives last (atomic ticket) reduces all partials in a
// fixed order; it resets the ticket for the next launch (graph replays).
__device__ __forceinline__ bool arrive_last_n(unsigned *counter, unsigned nblocks, int *sflag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(counter, 1u);
        TOPK_DCHECK(prev < nblocks, "last-block ticket past the grid (counter not reset)");
        *sflag = (prev == nblocks - 1);
    }
    __syncthreads();
    const bool last = *sflag;
    if (last) __threadfence();
    return last;
}
__device__ __forceinline__ bool arrive_last(unsigned *counter, int *sflag) {
    return arrive_last_n(counter, gridDim.x, sflag);
}

// ---- counter-based start vector (reading Q8) ---------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace topk
