// gather4_lab.cu -- can the TMA engine gather faster than the LSU/L1TEX path?
// The SpMV's x gathers run at ~1 distinct line per SM clock through LDG (the L1TEX tag
// stage, profiles/r02_spmv_bound.md). Blackwell's cp.async.bulk.tensor...tile::gather4
// fetches four 16-byte rows of a 2-D tensor at four arbitrary row coordinates into shared
// memory without the LSU. Here: 61M uniform random 4-byte gathers from a 4M-float
// (16.8 MB, L2-resident) vector, viewed as [n/4][4]; every thread issues one gather4 per
// step for its 4 indices into its own (128-byte aligned) shared slot, the CTA waits on an mbarrier
// (two stages), then each thread picks its 4 values out of shared memory and sums them.
// Compared with the LDG loop of tools/lab/tex_lab.cu (257-271 G gathers/s).
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/lab/gather4_lab.cu -o tools/lab/gather4_lab
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sptr(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sptr(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sptr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(sptr(b)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void gather4(void *dst, const CUtensorMap *map, int c0, int r0, int r1, int r2, int r3, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(
            sptr(dst)),
        "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sptr(bar))
        : "memory");
}

constexpr int NT = 128;  // 2 stages x 128 threads x 128-byte slots (TMA destinations are 128-byte aligned)
__global__ void __launch_bounds__(NT) kg4(const __grid_constant__ CUtensorMap map, const int *__restrict__ idx, int64_t N,
                                          float *out) {
    __shared__ alignas(128) float slot[2][NT][32];  // 64 bytes used per 128-byte slot
    __shared__ alignas(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    if (tid == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int64_t per_step = (int64_t)gridDim.x * NT * 4;  // gathers per grid step
    const int64_t steps = (N + per_step - 1) / per_step;
    float acc = 0.f;
    int cidx[2][4];
    auto issue = [&](int64_t s, int st) {
        const int64_t base = (s * gridDim.x + blockIdx.x) * (int64_t)NT * 4 + (int64_t)tid * 4;
        int r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t k = base + u;
            const int c = k < N ? __ldcs(idx + k) : 0;
            cidx[st][u] = c;
            r[u] = c >> 2;
        }
        if (tid == 0) mbar_expect(&bar[st], NT * 64);
        __syncthreads();  // expect_tx posted before any completion
        gather4(&slot[st][tid][0], &map, 0, r[0], r[1], r[2], r[3], &bar[st]);
    };
    unsigned phase[2] = {0, 0};
    if (steps > 0) issue(0, 0);
    for (int64_t s = 0; s < steps; ++s) {
        const int st = (int)(s & 1);
        if (s + 1 < steps) issue(s + 1, st ^ 1);
        mbar_wait(&bar[st], phase[st]);
        phase[st] ^= 1;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += slot[st][tid][4 * u + (cidx[st][u] & 3)];
        __syncthreads();  // slot[st] reusable
    }
    out[(int64_t)blockIdx.x * NT + tid] = acc;
}

__global__ void __launch_bounds__(NT) kldg(const int *__restrict__ idx, const float *__restrict__ x, int64_t N, float *out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    constexpr int U = 8;
    for (int64_t b = t; b < N; b += nt * U) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = (b + u * nt < N) ? __ldcs(idx + b + u * nt) : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) acc += __ldg(x + c[u]);
    }
    out[t] = acc;
}

int main() {
    const int64_t N = 61244826 / 1024 * 1024, n = 4194304;
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<int> hu(N);
    std::mt19937_64 rng(1);
    for (int64_t i = 0; i < N; ++i) hu[i] = (int)(rng() % n);
    int *du;
    float *dx, *dout;
    cudaMalloc(&du, N * 4); cudaMalloc(&dx, n * 4); cudaMalloc(&dout, (size_t)nsm * 16 * NT * 4);
    cudaMemcpy(du, hu.data(), N * 4, cudaMemcpyHostToDevice);
    std::vector<float> hx(n);
    for (int64_t i = 0; i < n; ++i) hx[i] = (float)(i % 97) * 0.25f;
    cudaMemcpy(dx, hx.data(), n * 4, cudaMemcpyHostToDevice);
    // tensor map: 2-D [n/4 rows][4 floats], box {4, 1}
    typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                                 const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
        printf("no cuTensorMapEncodeTiled\n");
        return 1;
    }
    CUtensorMap map;
    cuuint64_t dims[2] = {4, (cuuint64_t)(n / 4)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
    // reference sum
    double ref = 0;
    for (int64_t i = 0; i < N; ++i) ref += hx[hu[i]];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int bps : {1, 2, 4, 8}) {
        const int grid = nsm * bps;
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            kg4<<<grid, NT>>>(map, du, N, dout);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        cudaError_t err = cudaGetLastError();
        std::vector<float> ho((size_t)grid * NT);
        cudaMemcpy(ho.data(), dout, ho.size() * 4, cudaMemcpyDeviceToHost);
        double s = 0;
        for (float v : ho) s += v;
        printf("gather4 bps %d: %8.1f us  %6.1f G gathers/s  sum rel err %.2e  %s\n", bps, best * 1e3, N / (best * 1e-3) / 1e9,
               (s - ref) / ref, cudaGetErrorString(err));
    }
    for (int bps : {4, 8}) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            kldg<<<nsm * bps, NT>>>(du, dx, N, dout);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        printf("ldg     bps %d: %8.1f us  %6.1f G gathers/s\n", bps, best * 1e3, N / (best * 1e-3) / 1e9);
    }
    return 0;
}
