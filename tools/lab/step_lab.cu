// step_lab.cu — what limits the multi-dot (k_step shape) on B200: V has NC
// columns of n f32; each variant streams them once (dev tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int NC, int MODE>  // MODE 0: w loaded; 1: w = y - a u1 - b u0 (3 loads) + stored; 2: like 1 but columns predicated by it
__global__ void __launch_bounds__(256) k(const float *V, const float *y, float *w, int64_t n, int it, double *out) {
    double acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = 0;
    const int64_t nv = n / 4;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        uint4 u[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j)
            if (MODE < 2 || j < it) u[j] = __ldg(reinterpret_cast<const uint4 *>(V + j * n) + v);
        double ww[4];
        if (MODE == 0) {
            float4 t = __ldg(reinterpret_cast<const float4 *>(w) + v);
            ww[0] = t.x; ww[1] = t.y; ww[2] = t.z; ww[3] = t.w;
        } else {
            float4 a = __ldg(reinterpret_cast<const float4 *>(y) + v);
            float4 b = __ldg(reinterpret_cast<const float4 *>(V + (NC - 1) * n) + v);
            float4 c = __ldg(reinterpret_cast<const float4 *>(V + (NC - 2) * n) + v);
            ww[0] = a.x - 0.5 * b.x - 0.25 * c.x; ww[1] = a.y - 0.5 * b.y - 0.25 * c.y;
            ww[2] = a.z - 0.5 * b.z - 0.25 * c.z; ww[3] = a.w - 0.5 * b.w - 0.25 * c.w;
            float4 r = make_float4((float)ww[0], (float)ww[1], (float)ww[2], (float)ww[3]);
            reinterpret_cast<float4 *>(w)[v] = r;
            ww[0] = r.x; ww[1] = r.y; ww[2] = r.z; ww[3] = r.w;
        }
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            if (MODE < 2 || j < it) {
                const float *e = reinterpret_cast<const float *>(&u[j]);
                acc[j] += (double)e[0] * ww[0] + (double)e[1] * ww[1] + (double)e[2] * ww[2] + (double)e[3] * ww[3];
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < NC; ++j) s += acc[j];
    if (s == 12345.678) out[0] = s;
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int64_t n = 1 << 22;
    float *V, *y, *w; double *out;
    cudaMalloc(&V, 4 * n * 24); cudaMalloc(&y, 4 * n); cudaMalloc(&w, 4 * n); cudaMalloc(&out, 64);
    cudaMemset(V, 0, 4 * n * 24); cudaMemset(y, 0, 4 * n); cudaMemset(w, 0, 4 * n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char *name, auto kern, int bpsm, double bytes) {
        kern<<<nsm * bpsm, 256>>>(V, y, w, n, 17, out); cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) kern<<<nsm * bpsm, 256>>>(V, y, w, n, 17, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
        cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
        printf("%-44s regs %3d  %8.2f us  %6.0f GB/s (%s)\n", name, fa.numRegs, ms * 1e3, bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    const double B17w = 4.0 * n * 18, B17y = 4.0 * n * (17 + 1 + 1);
    for (int bpsm : {2, 4}) {
        printf("-- grid %d x 148\n", bpsm);
        run("NC=17 w loaded", k<17, 0>, bpsm, B17w);
        run("NC=17 w = f(y,u1,u0) stored", k<17, 1>, bpsm, B17y);
        run("NC=24 pred it=17, w computed+stored", k<24, 2>, bpsm, B17y);
        run("NC=16 pred it=17 (width 16)", k<16, 2>, bpsm, 4.0 * n * 18);
        run("NC=9 w loaded (half pass)", k<9, 0>, bpsm, 4.0 * n * 10);
    }
    return 0;
}
