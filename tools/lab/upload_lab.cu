// upload_lab.cu -- how fast can a host CSR (C3-sized: 245 MB int32 cols + 490 MB f64
// values, pageable caller memory) reach the device? (e2e create's floor)
//  1. cudaMemcpy straight from pageable memory (driver staging)
//  2. our staging: OpenMP memcpy into two 32 MB pinned buffers, DMA of chunk i
//     overlapping the fill of chunk i+1 (mem_pool.cpp staged_h2d), values as f64
//  3. the same with the f64 -> f32 rounding in the fill (what FDF uploads)
//  4. cudaHostRegister of the caller's arrays + one DMA each (+ unregister)
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fopenmp
//        tools/lab/upload_lab.cu -o tools/lab/upload_lab
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <omp.h>
#include <cuda_runtime.h>

static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

template <class Fill>
static void staged(void *dst, size_t bytes, char *buf[2], cudaStream_t st, Fill fill) {
    const size_t C = size_t(32) << 20;
    int b = 0;
    for (size_t off = 0; off < bytes; off += C, b ^= 1) {
        const size_t n = std::min(C, bytes - off);
        fill(buf[b], off, n);
        if (off > 0) cudaStreamSynchronize(st);
        cudaMemcpyAsync((char *)dst + off, buf[b], n, cudaMemcpyHostToDevice, st);
    }
    cudaStreamSynchronize(st);
}

int main() {
    const size_t nnz = 61244826;
    std::vector<int> col(nnz);
    std::vector<double> val(nnz);
#pragma omp parallel for
    for (size_t i = 0; i < nnz; ++i) { col[i] = (int)(i * 2654435761u % 4194304); val[i] = (double)(i % 128) / 128.0; }
    void *dcol, *dval;
    cudaMalloc(&dcol, nnz * 4);
    cudaMalloc(&dval, nnz * 8);
    char *buf[2];
    cudaHostAlloc((void **)&buf[0], 32 << 20, 0);
    cudaHostAlloc((void **)&buf[1], 32 << 20, 0);
    cudaStream_t st;
    cudaStreamCreate(&st);
    auto pmemcpy = [](char *d, const char *s, size_t n) {
        const int nt = omp_get_max_threads();
        const size_t per = (n + nt - 1) / nt;
#pragma omp parallel for
        for (int t = 0; t < nt; ++t) {
            const size_t a = (size_t)t * per;
            if (a < n) std::memcpy(d + a, s + a, std::min(per, n - a));
        }
    };
    printf("threads %d, bytes col %.0f MB val(f64) %.0f MB\n", omp_get_max_threads(), nnz * 4 / 1e6, nnz * 8 / 1e6);
    for (int rep = 0; rep < 3; ++rep) {
        double t0 = now();
        cudaMemcpy(dcol, col.data(), nnz * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(dval, val.data(), nnz * 8, cudaMemcpyHostToDevice);
        double t1 = now();
        staged(dcol, nnz * 4, buf, st, [&](char *d, size_t off, size_t n) { pmemcpy(d, (const char *)col.data() + off, n); });
        staged(dval, nnz * 8, buf, st, [&](char *d, size_t off, size_t n) { pmemcpy(d, (const char *)val.data() + off, n); });
        double t2 = now();
        staged(dcol, nnz * 4, buf, st, [&](char *d, size_t off, size_t n) { pmemcpy(d, (const char *)col.data() + off, n); });
        staged(dval, nnz * 4, buf, st, [&](char *d, size_t off, size_t n) {
            const size_t k0 = off / 4, cnt = n / 4;
            float *f = (float *)d;
#pragma omp parallel for
            for (size_t k = 0; k < cnt; ++k) f[k] = (float)val[k0 + k];
        });
        double t3 = now();
        cudaHostRegister(col.data(), nnz * 4, cudaHostRegisterDefault);
        cudaHostRegister(val.data(), nnz * 8, cudaHostRegisterDefault);
        double t4 = now();
        cudaMemcpyAsync(dcol, col.data(), nnz * 4, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(dval, val.data(), nnz * 8, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st);
        double t5 = now();
        cudaHostUnregister(col.data());
        cudaHostUnregister(val.data());
        double t6 = now();
        printf("rep %d: pageable cudaMemcpy %.1f ms (%.1f GB/s) | staged f64 %.1f ms (%.1f GB/s) | staged f32 vals %.1f ms | "
               "register %.1f ms + DMA %.1f ms (%.1f GB/s) + unregister %.1f ms\n",
               rep, (t1 - t0) * 1e3, nnz * 12 / (t1 - t0) / 1e9, (t2 - t1) * 1e3, nnz * 12 / (t2 - t1) / 1e9,
               (t3 - t2) * 1e3, (t4 - t3) * 1e3, (t5 - t4) * 1e3, nnz * 12 / (t5 - t4) / 1e9, (t6 - t5) * 1e3);
    }
    return 0;
}
