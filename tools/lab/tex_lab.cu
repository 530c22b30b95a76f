// tex_lab.cu -- is the random-gather line rate (~1 L1TEX tag lookup per SM clock,
// profiles/r02_spmv_bound.md) the same through the texture path? 61M uniform random
// 4-byte gathers from a 4M-float (16.8 MB, L2-resident) vector plus the int32 index
// stream, summed per thread: __ldg (LDG through L1) vs tex1Dfetch (TEX) vs ld.global.cg
// (L2 only), and the C3-like power-law index stream.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/lab/tex_lab.cu -o tools/lab/tex_lab
#include <cstdio>
#include <cmath>
#include <random>
#include <vector>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) kgather(const int *__restrict__ idx, const float *__restrict__ x,
                                               cudaTextureObject_t tex, int64_t N, float *out) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    constexpr int U = 8;
    for (int64_t b = tid; b < N; b += nt * U) {
        int c[U];
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = (b + u * nt < N) ? __ldcs(idx + b + u * nt) : 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float v;
            if (MODE == 0) v = __ldg(x + c[u]);
            else if (MODE == 1) v = tex1Dfetch<float>(tex, c[u]);
            else v = __ldcg(x + c[u]);
            acc += v;
        }
    }
    out[tid] = acc;
}

int main() {
    const int64_t N = 61244826, n = 4194304;
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<int> hu(N), hp(N);
    std::mt19937_64 rng(1);
    for (int64_t i = 0; i < N; ++i) hu[i] = (int)(rng() % n);
    std::uniform_real_distribution<double> U(0, 1);
    const double a = std::log(0.59) / std::log(57344.0 / n);
    for (int64_t i = 0; i < N; ++i) { int c = (int)(n * std::pow(U(rng), 1.0 / a)); hp[i] = c < n ? c : n - 1; }
    int *du, *dp;
    float *dx, *dout;
    cudaMalloc(&du, N * 4); cudaMalloc(&dp, N * 4); cudaMalloc(&dx, n * 4); cudaMalloc(&dout, (size_t)nsm * 8 * 256 * 4);
    cudaMemcpy(du, hu.data(), N * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, hp.data(), N * 4, cudaMemcpyHostToDevice);
    cudaMemset(dx, 0, n * 4);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = dx;
    rd.res.linear.desc = cudaCreateChannelDesc<float>();
    rd.res.linear.sizeInBytes = n * 4;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) { printf("texture create failed\n"); return 1; }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char *names[3] = {"ldg (L1)", "tex1Dfetch", "ld.cg (L2)"};
    for (int bps : {4, 8}) {
        const int grid = nsm * bps;
        for (int stream = 0; stream < 2; ++stream) {
            const int *ix = stream ? dp : du;
            for (int mode = 0; mode < 3; ++mode) {
                float best = 1e30f;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaEventRecord(e0);
                    if (mode == 0) kgather<0><<<grid, 256>>>(ix, dx, tex, N, dout);
                    else if (mode == 1) kgather<1><<<grid, 256>>>(ix, dx, tex, N, dout);
                    else kgather<2><<<grid, 256>>>(ix, dx, tex, N, dout);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    if (rep > 0 && ms < best) best = ms;
                }
                printf("bps %d %-9s %-11s %8.1f us  %6.1f G gathers/s\n", bps, stream ? "powerlaw" : "uniform", names[mode],
                       best * 1e3, N / (best * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
