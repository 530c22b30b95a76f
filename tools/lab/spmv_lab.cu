// spmv_lab.cu — isolate what bounds the SELL-32 SpMV on the real C3 physical
// layout (dev tool; inputs dumped by tools/lab/dump_c3.py). SELL items only
// (the big-row chunks are < 25% of nnz and handled separately).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <string>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <class T> std::vector<T> rd(const std::string &f) {
    FILE *fp = fopen(f.c_str(), "rb"); fseek(fp, 0, SEEK_END); long n = ftell(fp); fseek(fp, 0, SEEK_SET);
    std::vector<T> v(n / sizeof(T)); size_t got = fread(v.data(), 1, n, fp); (void)got; fclose(fp); return v;
}
// gather policies. P 0: plain ldg; 1: predicated evict_last (hot) / no_allocate (cold) on x;
// 2: predicated ld.shared (hot, smem index = c & mask) / ld.global no_allocate (cold);
// 3: predicated ld.shared (hot) / plain ldg (cold). Hot flag = bit 31 of c. x index = c & mask
// for P 0,1 (hot region = x prefix), smem index for P 2,3 (same value here: G = 1).
__constant__ int c_H;
template <int P>
__device__ __forceinline__ float gat(const float *x, const float *hot, int c) {
    float v;
    const unsigned idx = (unsigned)c & 0x7fffffffu;
    if (P == 0) return __ldg(x + idx);
    if (P == 8) return (float)(idx & 7);   // no gather at all (stream-only bound)
    if (P == 10) {  // position-based hybrid, predicated (no branch: both loads issue in the batch)
        const unsigned sa = (unsigned)__cvta_generic_to_shared(hot) + 4u * idx;
        asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2;\n\t"
                     "@p ld.shared.f32 %0, [%3];\n\t"
                     "@!p ld.global.nc.f32 %0, [%4];}"
                     : "=f"(v) : "r"(idx), "r"(c_H), "r"(sa), "l"(x + idx));
        return v;
    }
    if (P == 9) {  // position-based hybrid: hub prefix [0, H) from shared memory, the rest plain ldg
        return idx < (unsigned)c_H ? hot[idx] : __ldg(x + idx);
    }
    if (P == 6) return hot[idx % 51200u];  // all gathers from shared memory (throughput probe)
    if (P == 7) return hot[idx & 16383u];  // all gathers from a 64 KB smem window
    if (P == 4) {  // position-based: hub prefix [0, 65536) evict_last, the rest evict_first
        asm volatile("{.reg .pred p; setp.lt.u32 p, %1, 65536;\n\t"
                     "@p ld.global.nc.L1::evict_last.f32 %0, [%2];\n\t"
                     "@!p ld.global.nc.L1::evict_first.f32 %0, [%2];}"
                     : "=f"(v) : "r"(idx), "l"(x + idx));
        return v;
    }
    if (P == 5) {  // position-based: hub prefix normal, the rest evict_first
        asm volatile("{.reg .pred p; setp.lt.u32 p, %1, 65536;\n\t"
                     "@p ld.global.nc.f32 %0, [%2];\n\t"
                     "@!p ld.global.nc.L1::evict_first.f32 %0, [%2];}"
                     : "=f"(v) : "r"(idx), "l"(x + idx));
        return v;
    }
    if (P == 1) {
        asm volatile("{.reg .pred p; setp.lt.s32 p, %1, 0;\n\t"
                     "@p ld.global.nc.L1::evict_last.f32 %0, [%2];\n\t"
                     "@!p ld.global.nc.L1::no_allocate.f32 %0, [%2];}"
                     : "=f"(v) : "r"(c), "l"(x + idx));
        return v;
    }
    const unsigned sa = (unsigned)__cvta_generic_to_shared(hot + idx);
    if (P == 2)
        asm volatile("{.reg .pred p; setp.lt.s32 p, %1, 0;\n\t"
                     "@p ld.shared.f32 %0, [%2];\n\t"
                     "@!p ld.global.nc.L1::no_allocate.f32 %0, [%3];}"
                     : "=f"(v) : "r"(c), "r"(sa), "l"(x + idx));
    else
        asm volatile("{.reg .pred p; setp.lt.s32 p, %1, 0;\n\t"
                     "@p ld.shared.f32 %0, [%2];\n\t"
                     "@!p ld.global.nc.f32 %0, [%3];}"
                     : "=f"(v) : "r"(c), "r"(sa), "l"(x + idx));
    return v;
}
__device__ __forceinline__ int ldc(const int *p) { int v; asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
__device__ __forceinline__ float ldv(const float *p) { float v; asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v; }

// SELL items. P = gather policy (see gat); STREAM: 1 = no gathers (stream-only bound)
template <int P, int NT, int STREAM = 0, int MB = 1>
__global__ void __launch_bounds__(NT, MB) k(const int *col, const float *val, const int2 *sell, const int2 *items, int nitems,
                                        int nbig, int nne, const float *x, int H, double *y) {
    extern __shared__ float hot[];
    if (P == 2 || P == 3 || P == 6 || P == 7 || P == 9 || P == 10) {
        const int HH = (P == 7) ? 16384 : H;
        for (int i = threadIdx.x; i < HH; i += NT) hot[i] = x[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * NT + threadIdx.x) >> 5, nw = gridDim.x * NT / 32;
    constexpr int GQ = 8;
    for (int wi = gw; wi < nitems; wi += nw) {
        const int2 I = items[wi];
        const int base = sell[I.x].x;
        const int2 Sl = sell[I.y - 1];
        const int ntot = (Sl.x - base) / 32 + Sl.y;
        int sl = I.x, bound = sell[sl].y;
        double acc = 0;
        for (int t0 = 0; t0 < ntot; t0 += GQ) {
            int cc[GQ]; float vv[GQ], xg[GQ];
#pragma unroll
            for (int q = 0; q < GQ; ++q) {
                const int k = base + lane + 32 * (t0 + q);
                cc[q] = (t0 + q < ntot) ? ldc(col + k) : 0;
                vv[q] = (t0 + q < ntot) ? ldv(val + k) : 0.f;
            }
#pragma unroll
            for (int q = 0; q < GQ; ++q) xg[q] = STREAM ? (float)(cc[q] & 7) : gat<P>(x, hot, cc[q]);
#pragma unroll
            for (int q = 0; q < GQ; ++q) {
                const int t = t0 + q;
                if (t < ntot) {
                    acc += (double)vv[q] * (double)xg[q];
                    if (t + 1 == bound) {
                        const int row = nbig + 32 * sl + lane;
                        if (row < nne) y[row] = acc;
                        acc = 0; ++sl;
                        if (sl < I.y) bound += sell[sl].y;
                    }
                }
            }
        }
    }
}

// big-row chunks (rows of degree > 128, 72% of C3's nnz): warp per chunk
// V 0: scalar lanes k = zb + lane + 32t (product structure), 8 in flight
// V 1: 16-byte vectors: lane covers 4 consecutive nnz, aligned groups, masked ends
template <int V, int NT, int P = 0, int GQ = 8, int MB = 1>
__global__ void __launch_bounds__(NT, MB) kc(const int *col, const float *val, const int4 *chunks, int nch,
                                         const float *x, double *y, int H) {
    extern __shared__ float hot[];
    if (P == 2 || P == 3 || P == 6 || P == 7 || P == 9 || P == 10) {
        const int HH = (P == 7) ? 16384 : H;
        for (int i = threadIdx.x; i < HH; i += NT) hot[i] = x[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * NT + threadIdx.x) >> 5, nw = gridDim.x * NT / 32;
    for (int wi = gw; wi < nch; wi += nw) {
        const int4 C = chunks[wi];
        const int zb = C.y, ze = C.y + C.z;
        double acc = 0;
        if (V == 0) {
            for (int k0 = zb + lane; k0 < ze; k0 += 32 * GQ) {
                int cc[GQ]; float vv[GQ];
#pragma unroll
                for (int q = 0; q < GQ; ++q) { const int k = k0 + 32 * q; cc[q] = k < ze ? ldc(col + k) : 0; vv[q] = k < ze ? ldv(val + k) : 0.f; }
#pragma unroll
                for (int q = 0; q < GQ; ++q) acc += (double)vv[q] * (double)gat<P>(x, hot, cc[q]);
            }
        } else {
            const int z4 = zb & ~3;
            constexpr int GQ = 4;  // 4 vectors of 4 = 16 nnz per lane per group
            for (int k0 = z4 + 4 * lane; k0 < ze; k0 += 128 * GQ) {
                int4 c4[GQ]; float4 v4[GQ];
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    const int k = k0 + 128 * q;
                    if (k < ze) {
                        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(c4[q].x), "=r"(c4[q].y), "=r"(c4[q].z), "=r"(c4[q].w) : "l"(col + k));
                        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v4[q].x), "=f"(v4[q].y), "=f"(v4[q].z), "=f"(v4[q].w) : "l"(val + k));
                    } else { c4[q] = make_int4(0, 0, 0, 0); v4[q] = make_float4(0, 0, 0, 0); }
                }
#pragma unroll
                for (int q = 0; q < GQ; ++q) {
                    const int k = k0 + 128 * q;
                    const int cc[4] = {c4[q].x, c4[q].y, c4[q].z, c4[q].w};
                    const float vv[4] = {v4[q].x, v4[q].y, v4[q].z, v4[q].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (k + e >= zb && k + e < ze) acc += (double)vv[e] * (double)gat<P>(x, hot, cc[e]);
                }
            }
        }
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) y[wi] = acc;
    }
}

int main(int argc, char **argv) {
    std::string d = argc > 1 ? argv[1] : "/tmp/c3";
    auto pcol = rd<int>(d + "/pcol.bin"); auto pval = rd<float>(d + "/pval.bin");
    auto sell = rd<int>(d + "/sell.bin"); auto items = rd<int>(d + "/items.bin"); auto meta = rd<long long>(d + "/meta.bin");
    const int nbig = (int)meta[0], nne = (int)meta[1], n = (int)meta[2], H = (int)meta[3];
    int *dcol; float *dval; int2 *dsell, *ditems; float *dx; double *dy;
    CK(cudaMalloc(&dcol, pcol.size() * 4 + 512)); CK(cudaMalloc(&dval, pval.size() * 4 + 512));
    CK(cudaMalloc(&dsell, sell.size() * 4)); CK(cudaMalloc(&ditems, items.size() * 4));
    CK(cudaMalloc(&dx, (size_t)n * 4)); CK(cudaMalloc(&dy, (size_t)n * 8));
    cudaMemcpy(dcol, pcol.data(), pcol.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dval, pval.data(), pval.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dsell, sell.data(), sell.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(ditems, items.data(), items.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dx, 0, (size_t)n * 4);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int nitems = (int)items.size() / 2;
    long long sellnnz = (long long)pcol.size() - 0;
    printf("nbig %d nne %d n %d H %d nitems %d phys %zu\n", nbig, nne, n, H, nitems, pcol.size());
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int Hs = H;
    auto setH = [&](int h) { Hs = h; cudaMemcpyToSymbol(c_H, &h, 4); };
    auto attr = [&](auto kern) { cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern); return fa.numRegs; };
    auto run = [&](const char *name, auto kern, int nt, int bpsm, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nsm * bpsm, nt, smem>>>(dcol, dval, dsell, ditems, nitems, nbig, nne, dx, Hs, dy);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) kern<<<nsm * bpsm, nt, smem>>>(dcol, dval, dsell, ditems, nitems, nbig, nne, dx, Hs, dy);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
        printf("%-40s H %6d regs %3d %8.3f us   (%s)\n", name, Hs, attr(kern), ms * 1e3, cudaGetErrorString(cudaGetLastError()));
    };
    setH(H);
    run("SELL P0 ldg 256x3", k<0, 256>, 256, 3, 0);
    run("SELL P0 ldg 256x4 mb4", k<0, 256, 0, 4>, 256, 4, 0);
    run("SELL P0 ldg 256x5 mb5", k<0, 256, 0, 5>, 256, 5, 0);
    run("SELL P0 ldg 256x6 mb6", k<0, 256, 0, 6>, 256, 6, 0);
    run("SELL P6 all-smem 1024x1", k<6, 1024>, 1024, 1, (size_t)H * 4);
    setH(51200); run("SELL P10 pred-hybrid 768x1", k<10, 768>, 768, 1, 51200 * 4);
    setH(51200); run("SELL P10 pred-hybrid 1024x1", k<10, 1024>, 1024, 1, 51200 * 4);
    setH(27648); run("SELL P10 pred-hybrid 384x2", k<10, 384, 0, 2>, 384, 2, 27648 * 4);
    setH(27648); run("SELL P10 pred-hybrid 512x2", k<10, 512, 0, 2>, 512, 2, 27648 * 4);
    setH(18432); run("SELL P10 pred-hybrid 256x3", k<10, 256, 0, 3>, 256, 3, 18432 * 4);
    setH(13824); run("SELL P10 pred-hybrid 256x4", k<10, 256, 0, 4>, 256, 4, 13824 * 4);
    setH(8192); run("SELL P10 pred-hybrid 256x4 H8k", k<10, 256, 0, 4>, 256, 4, 8192 * 4);
    setH(H);
    auto bcol = rd<int>(d + "/bcol.bin"); auto bval = rd<float>(d + "/bval.bin"); auto ch = rd<int>(d + "/chunks.bin");
    int *dbc; float *dbv; int4 *dch;
    CK(cudaMalloc(&dbc, bcol.size() * 4 + 4096)); CK(cudaMalloc(&dbv, bval.size() * 4 + 4096)); CK(cudaMalloc(&dch, ch.size() * 4));
    cudaMemcpy(dbc, bcol.data(), bcol.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dbv, bval.data(), bval.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dch, ch.data(), ch.size() * 4, cudaMemcpyHostToDevice);
    const int nch = (int)ch.size() / 4;
    printf("big rows: nnz %zu chunks %d\n", bcol.size(), nch);
    auto runc = [&](const char *name, auto kern, int nt, int bpsm, size_t smem = 0) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<nsm * bpsm, nt, smem>>>(dbc, dbv, dch, nch, dx, dy, Hs);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) kern<<<nsm * bpsm, nt, smem>>>(dbc, dbv, dch, nch, dx, dy, Hs);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
        printf("%-40s H %6d regs %3d %8.3f us  %.0f GB/s algorithmic (%s)\n", name, Hs, attr(kern), ms * 1e3, bcol.size() * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    runc("chunks scalar P0 256x3", kc<0, 256, 0>, 256, 3);
    runc("chunks scalar P0 256x4 mb4", kc<0, 256, 0, 8, 4>, 256, 4);
    runc("chunks scalar P8 stream-only 256x3", kc<0, 256, 8>, 256, 3);
    setH(51200); runc("chunks P10 pred-hybrid 768x1", kc<0, 768, 10>, 768, 1, 51200 * 4);
    setH(51200); runc("chunks P10 pred-hybrid 1024x1", kc<0, 1024, 10>, 1024, 1, 51200 * 4);
    setH(27648); runc("chunks P10 pred-hybrid 384x2", kc<0, 384, 10, 8, 2>, 384, 2, 27648 * 4);
    setH(27648); runc("chunks P10 pred-hybrid 512x2", kc<0, 512, 10, 8, 2>, 512, 2, 27648 * 4);
    setH(18432); runc("chunks P10 pred-hybrid 256x3", kc<0, 256, 10, 8, 3>, 256, 3, 18432 * 4);
    setH(13824); runc("chunks P10 pred-hybrid 256x4", kc<0, 256, 10, 8, 4>, 256, 4, 13824 * 4);
    setH(8192); runc("chunks P10 pred-hybrid 256x4 H8k", kc<0, 256, 10, 8, 4>, 256, 4, 8192 * 4);
    runc("chunks scalar P0 256x5 mb5", kc<0, 256, 0, 8, 5>, 256, 5);
    runc("chunks scalar P0 256x6 mb6", kc<0, 256, 0, 8, 6>, 256, 6);
    setH(51200); runc("chunks scalar P6 all-smem 1024x1", kc<0, 1024, 6>, 1024, 1, 51200 * 4);
    return 0;
}
