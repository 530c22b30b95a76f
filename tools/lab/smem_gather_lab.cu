// smem_gather_lab.cu -- can a streaming SpMV pass with shared-memory x gathers run at
// HBM speed on B200? 40 M entries (u16 index into a 57,344-entry f32 x staged in shared
// memory once per CTA, f32 value), per-warp contiguous ranges (interleaved physical
// layout, see layout_lab.cu), fp64 accumulation. Variants: CTA size / CTAs per SM /
// prefetch depth; index distribution uniform or power-law (C3-like hub skew).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cmath>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int H = 57344;

template <int GQ, int NT, int MB, int SMEM_X>
__global__ void __launch_bounds__(NT, MB) khub(const uint16_t *col, const float *val, const float *x, int64_t T, int W,
                                               double *out) {
    extern __shared__ float xs[];
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * NT + threadIdx.x) >> 5;
    const int HH = SMEM_X ? H : 1;
    for (int i = threadIdx.x; i < HH; i += NT) xs[i] = x[i];
    __syncthreads();
    if (w >= W) return;
    auto gidx = [&](int64_t j) -> int64_t { return j * W + w; };
    int cc[GQ]; float vv[GQ];
#pragma unroll
    for (int q = 0; q < GQ; ++q) { int64_t k = gidx(q) * 32 + lane; cc[q] = __ldcs(col + k); vv[q] = __ldcs(val + k); }
    double acc = 0;
    for (int64_t j = 0; j < T; j += GQ) {
        float xg[GQ];
#pragma unroll
        for (int q = 0; q < GQ; ++q) xg[q] = SMEM_X ? xs[cc[q]] : __ldg(x + cc[q]);
        float vc[GQ];
#pragma unroll
        for (int q = 0; q < GQ; ++q) {
            vc[q] = vv[q];
            int64_t jn = j + GQ + q;
            if (jn < T) { int64_t k = gidx(jn) * 32 + lane; cc[q] = __ldcs(col + k); vv[q] = __ldcs(val + k); }
        }
#pragma unroll
        for (int q = 0; q < GQ; ++q) acc += (double)vc[q] * (double)xg[q];
    }
    out[w * 32 + lane] = acc;
}

int main() {
    const int64_t N = 40000000 / 32 * 32;
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<uint16_t> hu(N), hp(N);
    std::mt19937_64 rng(1);
    std::uniform_real_distribution<double> U(0, 1);
    for (int64_t i = 0; i < N; ++i) hu[i] = (uint16_t)(rng() % H);
    for (int64_t i = 0; i < N; ++i) { int c = (int)(H * std::pow(U(rng), 3.0)); hp[i] = (uint16_t)(c < H ? c : H - 1); }
    uint16_t *du, *dp; float *dv, *dx; double *dout;
    CK(cudaMalloc(&du, N * 2)); CK(cudaMalloc(&dp, N * 2)); CK(cudaMalloc(&dv, N * 4)); CK(cudaMalloc(&dx, H * 4));
    CK(cudaMalloc(&dout, 1 << 24));
    CK(cudaMemcpy(du, hu.data(), N * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, hp.data(), N * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(dv, 0, N * 4)); CK(cudaMemset(dx, 0, H * 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char *name, auto kern, int nt, int bps, bool smem, const uint16_t *colp) {
        const size_t sm = smem ? H * 4 : 0;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const int W = nsm * bps * nt / 32;
        const int64_t T = (N / 32) / W;
        kern<<<nsm * bps, nt, sm>>>(colp, dv, dx, T, W, dout);
        cudaEventRecord(e0);
        for (int r = 0; r < 10; ++r) kern<<<nsm * bps, nt, sm>>>(colp, dv, dx, T, W, dout);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)T * W * 32 * 6;
        printf("%-40s %8.1f us  %6.0f GB/s (6 B/entry)  %s\n", name, ms * 100, bytes / (ms * 1e-4) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("smem uniform 1024x1 GQ8", khub<8, 1024, 1, 1>, 1024, 1, true, du);
    run("smem uniform 1024x1 GQ4", khub<4, 1024, 1, 1>, 1024, 1, true, du);
    run("smem uniform 1024x1 GQ16", khub<16, 1024, 1, 1>, 1024, 1, true, du);
    run("smem powerlaw 1024x1 GQ8", khub<8, 1024, 1, 1>, 1024, 1, true, dp);
    run("smem uniform 512x1 GQ16", khub<16, 512, 1, 1>, 512, 1, true, du);
    run("smem uniform 768x1 GQ8", khub<8, 768, 1, 1>, 768, 1, true, du);
    run("stream only (x[0]) 1024x1 GQ8", khub<8, 1024, 1, 0>, 1024, 1, false, du);
    run("L1 gathers (no smem) 256x4 GQ8", khub<8, 256, 4, 0>, 256, 4, false, du);
    CK(cudaGetLastError());
    return 0;
}
