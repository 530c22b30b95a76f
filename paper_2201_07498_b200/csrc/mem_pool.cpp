// mem_pool.cpp — see mem_pool.h.
#include "mem_pool.h"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <unordered_map>
#include <utility>

#include <cstdlib>
#include <new>
#include <vector>

#include <omp.h>
#include <sys/mman.h>

namespace topk {

namespace {

struct DevPool {
    std::mutex mu;
    std::unordered_map<void *, std::pair<int, size_t>> live;  // ptr -> (device, size)
    std::multimap<std::pair<int, size_t>, void *> cached;      // (device, size) -> ptr
};
DevPool &dev_pool() {
    static DevPool *p = new DevPool();  // never destroyed: blocks may outlive static teardown
    return *p;
}

size_t round_size(size_t b) {
    if (b < (1u << 20)) return (b + 511) & ~size_t(511);
    const size_t g = size_t(2) << 20;
    return (b + g - 1) / g * g;
}

size_t trim_device_locked(DevPool &P, int dev) {
    size_t freed = 0;
    int cur = -1;
    cudaGetDevice(&cur);
    for (auto it = P.cached.begin(); it != P.cached.end();) {
        if (dev >= 0 && it->first.first != dev) { ++it; continue; }
        cudaSetDevice(it->first.first);
        cudaFree(it->second);
        freed += it->first.second;
        it = P.cached.erase(it);
    }
    if (cur >= 0) cudaSetDevice(cur);
    return freed;
}

}  // namespace

void *pool_dev_alloc(size_t bytes) {
    DevPool &P = dev_pool();
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    const size_t rb = round_size(std::max<size_t>(bytes, 256));
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.cached.lower_bound({dev, rb});
    if (it != P.cached.end() && it->first.first == dev && it->first.second <= rb + std::max(rb / 8, size_t(2) << 20)) {
        void *p = it->second;
        const size_t sz = it->first.second;
        P.cached.erase(it);
        P.live[p] = {dev, sz};
        return p;
    }
    void *p = nullptr;
    if (cudaMalloc(&p, rb) != cudaSuccess) {
        cudaGetLastError();
        trim_device_locked(P, dev);
        if (cudaMalloc(&p, rb) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
    }
    P.live[p] = {dev, rb};
    return p;
}

void pool_dev_free(void *p) {
    if (!p) return;
    DevPool &P = dev_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    auto it = P.live.find(p);
    if (it == P.live.end()) return;
    P.cached.insert({it->second, p});
    P.live.erase(it);
}

namespace {
struct HostPool {
    std::mutex mu;
    std::multimap<size_t, void *> cached;  // rounded size -> block
    size_t cached_bytes = 0;
};
HostPool &host_pool() {
    static HostPool *p = new HostPool();
    return *p;
}
constexpr size_t kHostGran = size_t(2) << 20;
constexpr size_t kHostCacheMax = size_t(8) << 30;  // cached (unused) host bytes kept at most
size_t host_round(size_t b) { return (b + kHostGran - 1) / kHostGran * kHostGran; }
size_t trim_host_locked(HostPool &P) {
    size_t freed = 0;
    for (auto &kv : P.cached) {
        std::free(kv.second);
        freed += kv.first;
    }
    P.cached.clear();
    P.cached_bytes = 0;
    return freed;
}
}  // namespace

void *host_block_alloc(size_t bytes) {
    const size_t rb = host_round(std::max<size_t>(bytes, 1));
    HostPool &P = host_pool();
    {
        std::lock_guard<std::mutex> lk(P.mu);
        auto it = P.cached.find(rb);
        if (it != P.cached.end()) {
            void *p = it->second;
            P.cached.erase(it);
            P.cached_bytes -= rb;
            return p;
        }
    }
    void *p = std::aligned_alloc(kHostGran, rb);
    if (!p) {
        {
            std::lock_guard<std::mutex> lk(P.mu);
            trim_host_locked(P);
        }
        p = std::aligned_alloc(kHostGran, rb);
        if (!p) throw std::bad_alloc();
    }
    madvise(p, rb, MADV_HUGEPAGE);  // advisory: fewer, larger first-touch faults
    return p;
}

void host_block_free(void *p, size_t bytes) {
    if (!p) return;
    const size_t rb = host_round(std::max<size_t>(bytes, 1));
    HostPool &P = host_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.cached_bytes + rb > kHostCacheMax) {
        std::free(p);
        return;
    }
    P.cached.insert({rb, p});
    P.cached_bytes += rb;
}

size_t pool_trim() {
    size_t freed = 0;
    {
        HostPool &H = host_pool();
        std::lock_guard<std::mutex> lk(H.mu);
        freed += trim_host_locked(H);
    }
    DevPool &P = dev_pool();
    std::lock_guard<std::mutex> lk(P.mu);
    return freed + trim_device_locked(P, -1);
}

void par_memcpy(void *dst, const void *src, size_t bytes) {
    if (bytes < (size_t(4) << 20)) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const int nt = omp_get_max_threads();
    const size_t per = (bytes + nt - 1) / nt;
#pragma omp parallel for schedule(static)
    for (int t = 0; t < nt; ++t) {
        const size_t a = (size_t)t * per;
        if (a >= bytes) continue;
        std::memcpy((char *)dst + a, (const char *)src + a, std::min(per, bytes - a));
    }
}

namespace {
constexpr size_t kStage = size_t(32) << 20;  // bytes per pinned chunk
struct Stage {
    std::mutex mu;
    char *buf[2] = {nullptr, nullptr};
};
Stage &stage() {
    static Stage *s = new Stage();
    return *s;
}
cudaError_t stage_buffers(Stage &S) {
    for (int b = 0; b < 2; ++b)
        if (!S.buf[b]) {
            cudaError_t e = cudaHostAlloc((void **)&S.buf[b], kStage, cudaHostAllocPortable);
            if (e != cudaSuccess) { S.buf[b] = nullptr; return e; }
        }
    return cudaSuccess;
}
}  // namespace

cudaError_t staged_h2d(void *dst_dev, size_t bytes, const StageFill &fill, cudaStream_t stream) {
    if (bytes == 0) return cudaSuccess;
    Stage &S = stage();
    std::lock_guard<std::mutex> lk(S.mu);
    cudaError_t e = stage_buffers(S);
    if (e != cudaSuccess) return e;
    // fill chunk i into buffer i % 2 while the DMA of chunk i - 1 runs
    int b = 0;
    for (size_t off = 0; off < bytes; off += kStage, b ^= 1) {
        const size_t n = std::min(kStage, bytes - off);
        fill(S.buf[b], off, n);
        if (off > 0 && (e = cudaStreamSynchronize(stream)) != cudaSuccess) return e;  // chunk i - 2's buffer free
        e = cudaMemcpyAsync((char *)dst_dev + off, S.buf[b], n, cudaMemcpyHostToDevice, stream);
        if (e != cudaSuccess) return e;
    }
    return cudaStreamSynchronize(stream);
}

cudaError_t staged_d2h(const void *src_dev, size_t bytes, const StageDrain &drain, cudaStream_t stream) {
    if (bytes == 0) return cudaSuccess;
    Stage &S = stage();
    std::lock_guard<std::mutex> lk(S.mu);
    cudaError_t e = stage_buffers(S);
    if (e != cudaSuccess) return e;
    size_t n0 = std::min(kStage, bytes);
    if ((e = cudaMemcpyAsync(S.buf[0], src_dev, n0, cudaMemcpyDeviceToHost, stream)) != cudaSuccess) return e;
    int b = 0;
    for (size_t off = 0; off < bytes; off += kStage, b ^= 1) {
        const size_t n = std::min(kStage, bytes - off);
        if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return e;  // chunk i landed
        const size_t off2 = off + kStage;
        if (off2 < bytes) {  // DMA of chunk i + 1 overlaps the drain of chunk i
            const size_t n2 = std::min(kStage, bytes - off2);
            e = cudaMemcpyAsync(S.buf[b ^ 1], (const char *)src_dev + off2, n2, cudaMemcpyDeviceToHost, stream);
            if (e != cudaSuccess) return e;
        }
        drain(S.buf[b], off, n);
    }
    return cudaStreamSynchronize(stream);
}

}  // namespace topk
