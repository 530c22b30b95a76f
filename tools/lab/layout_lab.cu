// layout_lab.cu -- does the per-warp stream layout matter? 61M (col int32, val f32)
// entries in 32-entry groups; each warp sums T consecutive groups of ITS stream.
//  mode 0: warp w's groups are physically contiguous [w T, (w+1) T)
//  mode 1: warp w's j-th group is physical group j W + w (warp-interleaved)
// gathers: 0 none (stream only), 1 x[col] from a 4M f32 vector (uniform random cols),
//          2 x[col] with col drawn from a power law (C3-like: 59% of entries in the
//          57K lowest indices)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int GQ, int MODE, int GATHER>
__global__ void __launch_bounds__(256) kstream(const int *col, const float *val, const float *x, int64_t T, int W, double *out) {
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * 256 + threadIdx.x) >> 5;
    if (w >= W) return;
    auto gidx = [&](int64_t j) -> int64_t { return MODE == 0 ? (int64_t)w * T + j : j * W + w; };
    int cc[GQ]; float vv[GQ];
#pragma unroll
    for (int q = 0; q < GQ; ++q) { int64_t k = gidx(q) * 32 + lane; cc[q] = __ldcs(col + k); vv[q] = __ldcs(val + k); }
    double acc = 0;
    for (int64_t j = 0; j < T; j += GQ) {
        float xg[GQ];
#pragma unroll
        for (int q = 0; q < GQ; ++q) xg[q] = GATHER ? __ldg(x + cc[q]) : (float)(cc[q] & 7);
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
    const int64_t N = 61244826 / 32 * 32, n = 4194304;
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<int> hc(N), hp(N);
    std::mt19937_64 rng(1);
    for (int64_t i = 0; i < N; ++i) hc[i] = (int)(rng() % n);
    // power law: P(col < c) ~ (c / n)^0.25-ish fitted so that 59% of draws fall below 57344
    std::uniform_real_distribution<double> U(0, 1);
    const double a = std::log(0.59) / std::log(57344.0 / n);
    for (int64_t i = 0; i < N; ++i) { int c = (int)(n * std::pow(U(rng), 1.0 / a)); hp[i] = c < n ? c : n - 1; }
    int *dc, *dp; float *dv, *dx; double *dout;
    CK(cudaMalloc(&dc, N * 4)); CK(cudaMalloc(&dp, N * 4)); CK(cudaMalloc(&dv, N * 4)); CK(cudaMalloc(&dx, n * 4));
    CK(cudaMalloc(&dout, 1 << 24));
    CK(cudaMemcpy(dc, hc.data(), N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, hp.data(), N * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(dv, 0, N * 4)); CK(cudaMemset(dx, 0, n * 4));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int bps : {2, 3, 4}) {
        const int W = nsm * bps * 8;
        const int64_t T = (N / 32 + W - 1) / W;
        auto run = [&](const char *name, auto kern, const int *colp) {
            kern<<<nsm * bps, 256>>>(colp, dv, dx, T - 1, W, dout);
            cudaEventRecord(e0);
            for (int r = 0; r < 10; ++r) kern<<<nsm * bps, 256>>>(colp, dv, dx, T - 1, W, dout);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("bps %d %-34s %8.1f us  %6.0f GB/s stream\n", bps, name, ms * 100, (double)(T - 1) * W * 32 * 8 / (ms * 1e-4) / 1e9);
        };
        run("contig  stream-only GQ8", kstream<8, 0, 0>, dc);
        run("interlv stream-only GQ8", kstream<8, 1, 0>, dc);
        run("contig  uniform-gather GQ8", kstream<8, 0, 1>, dc);
        run("interlv uniform-gather GQ8", kstream<8, 1, 1>, dc);
        run("contig  powerlaw-gather GQ8", kstream<8, 0, 1>, dp);
        run("interlv powerlaw-gather GQ8", kstream<8, 1, 1>, dp);
        run("interlv powerlaw-gather GQ4", kstream<4, 1, 1>, dp);
        run("interlv powerlaw-gather GQ16", kstream<16, 1, 1>, dp);
    }
    CK(cudaGetLastError());
    return 0;
}
