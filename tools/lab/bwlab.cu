// bwlab.cu — B200 memory-pattern ceilings for the hot path's kernels (dev tool,
// not part of the product): stream copy, multi-column read (multi-dot shape),
// random 4-byte gathers from an L2-resident vector (SpMV x gathers).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o bwlab bwlab.cu && ./bwlab
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_copy(const float4 *a, float4 *b, int64_t n4) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
// NC columns of n floats; thread = one float4 row-vector, all NC columns, NA accumulators
template <int NC>
__global__ void k_multidot(const float *V, int64_t n, const float *w, double *out) {
    double acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = 0;
    const int64_t nv = n / 4;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        float4 ww = __ldg(reinterpret_cast<const float4 *>(w) + v);
        float4 u[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) u[j] = __ldg(reinterpret_cast<const float4 *>(V + j * n) + v);
#pragma unroll
        for (int j = 0; j < NC; ++j) acc[j] += (double)u[j].x * ww.x + (double)u[j].y * ww.y + (double)u[j].z * ww.z + (double)u[j].w * ww.w;
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < NC; ++j) s += acc[j];
    if (s == 12345.678) out[0] = s;
}
// gathers: idx stream (int4) + x gathers; mode 0 ldg, 1 no_allocate, 2 evict_last if idx < H
template <int MODE>
__global__ void k_gather(const int *idx, int64_t m, const float *x, int H, double *out) {
    double s = 0;
    const int64_t m4 = m / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m4; i += (int64_t)gridDim.x * blockDim.x) {
        int4 c = __ldcs(reinterpret_cast<const int4 *>(idx) + i);
        int cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float v;
            const float *p = x + cc[e];
            if (MODE == 0) v = __ldg(p);
            else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
            else {
                if (cc[e] < H) asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p));
                else asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
            }
            s += v;
        }
    }
    if (s == 12345.678) out[0] = s;
}

template <typename F>
float timeit(F f, int reps = 10) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int64_t n = 1 << 22;  // 4.19M (C3)
    float *V, *w, *x, *big0, *big1; int *idx; double *out;
    const int NCmax = 24;
    CK(cudaMalloc(&V, sizeof(float) * n * NCmax)); CK(cudaMalloc(&w, sizeof(float) * n));
    CK(cudaMalloc(&x, sizeof(float) * n)); CK(cudaMalloc(&out, 64));
    const int64_t nb = 1ll << 28; CK(cudaMalloc(&big0, 4 * nb)); CK(cudaMalloc(&big1, 4 * nb));
    cudaMemset(V, 0, sizeof(float) * n * NCmax); cudaMemset(w, 0, 4 * n); cudaMemset(x, 0, 4 * n);
    cudaMemset(big0, 0, 4 * nb); cudaMemset(big1, 0, 4 * nb);
    // copy
    for (int bpsm : {4, 8}) {
        float ms = timeit([&] { k_copy<<<nsm * bpsm, 256>>>((float4 *)big0, (float4 *)big1, nb / 4); });
        printf("copy 1 GiB bpsm=%d: %.3f ms  %.0f GB/s (read+write)\n", bpsm, ms, 8.0 * nb / ms / 1e6);
    }
    // multi-dot
    for (int bpsm : {2, 4, 8}) {
        float ms = timeit([&] { k_multidot<8><<<nsm * bpsm, 256>>>(V, n, w, out); });
        printf("multidot NC=8  bpsm=%d: %.3f ms  %.0f GB/s\n", bpsm, ms, 4.0 * n * 9 / ms / 1e6);
        ms = timeit([&] { k_multidot<16><<<nsm * bpsm, 256>>>(V, n, w, out); });
        printf("multidot NC=16 bpsm=%d: %.3f ms  %.0f GB/s\n", bpsm, ms, 4.0 * n * 17 / ms / 1e6);
        ms = timeit([&] { k_multidot<24><<<nsm * bpsm, 256>>>(V, n, w, out); });
        printf("multidot NC=24 bpsm=%d: %.3f ms  %.0f GB/s\n", bpsm, ms, 4.0 * n * 25 / ms / 1e6);
    }
    // gathers: m = 61M indices, uniform random and zipf-like (power law, hubs first)
    const int64_t m = 61244826 / 4 * 4;
    std::vector<int> h(m);
    std::mt19937_64 rng(1);
    for (int64_t i = 0; i < m; ++i) h[i] = (int)(rng() % n);
    CK(cudaMalloc(&idx, 4 * m));
    cudaMemcpy(idx, h.data(), 4 * m, cudaMemcpyHostToDevice);
    for (int bpsm : {4, 8}) {
        float ms0 = timeit([&] { k_gather<0><<<nsm * bpsm, 256>>>(idx, m, x, 0, out); });
        float ms1 = timeit([&] { k_gather<1><<<nsm * bpsm, 256>>>(idx, m, x, 0, out); });
        printf("uniform gathers bpsm=%d: ldg %.3f ms (%.0f Ggather/s), no_alloc %.3f ms (%.0f Ggather/s)\n", bpsm, ms0,
               m / ms0 / 1e6, ms1, m / ms1 / 1e6);
    }
    // power-law: P(rank r) ~ r^-0.9 approx via inverse CDF on a continuous power law
    std::uniform_real_distribution<double> U(0, 1);
    for (int64_t i = 0; i < m; ++i) {
        double u = U(rng);
        double r = std::pow(u, 1.0 / 0.22) * n;  // heavy concentration at small ranks
        h[i] = std::min<int64_t>((int64_t)r, n - 1);
    }
    std::vector<int> hs(h.begin(), h.end()); std::sort(hs.begin(), hs.end());
    printf("power-law sample: share of gathers to rank < 49152: %.3f\n",
           (double)(std::lower_bound(hs.begin(), hs.end(), 49152) - hs.begin()) / m);
    cudaMemcpy(idx, h.data(), 4 * m, cudaMemcpyHostToDevice);
    for (int bpsm : {4, 8}) {
        float ms0 = timeit([&] { k_gather<0><<<nsm * bpsm, 256>>>(idx, m, x, 0, out); });
        float ms1 = timeit([&] { k_gather<1><<<nsm * bpsm, 256>>>(idx, m, x, 0, out); });
        float ms2 = timeit([&] { k_gather<2><<<nsm * bpsm, 256>>>(idx, m, x, 49152, out); });
        float ms3 = timeit([&] { k_gather<2><<<nsm * bpsm, 256>>>(idx, m, x, 24576, out); });
        printf("powerlaw gathers bpsm=%d: ldg %.3f ms, no_alloc %.3f ms, hot49k %.3f ms, hot24k %.3f ms (%.0f Ggather/s best)\n",
               bpsm, ms0, ms1, ms2, ms3, m / std::min(std::min(ms0, ms1), std::min(ms2, ms3)) / 1e6);
    }
    CK(cudaGetLastError());
    return 0;
}
