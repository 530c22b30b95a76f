// mem_pool.h — process-wide memory runtime of libtopk_eig (native, thread-safe):
//  * a caching device allocator: blocks freed by topk_eig_destroy go to a per-device
//    free list and are reused by the next topk_eig_create (no cudaMalloc/cudaFree
//    on the create/destroy path after the first handle; topk_eig_trim_pool() returns
//    the cached blocks to the driver);
//  * a caching host allocator for large blocks (>= 1 MB; the host-side layout arrays of
//    topk_eig_create): freed blocks are kept and reused, new ones are 2 MB aligned with
//    transparent huge pages requested, so repeated creates do not pay a page fault per
//    4 KB of fresh memory (measured on C3: 120 -> ~80 ms per create); at most 8 GB
//    of unused blocks are kept;
//  * staged host<->device copies through two pinned chunks: the host side of chunk
//    i+1 (a parallel memcpy or an element conversion) overlaps the DMA of chunk i,
//    so pageable caller buffers and the host-side layout move at pinned-copy speed.
#pragma once
#include <cstddef>
#include <cstdint>
#include <functional>

#include <cuda_runtime.h>

namespace topk {

// Device allocation on the current device. Returns nullptr on failure (the cache
// is trimmed and cudaMalloc retried once first).
void *pool_dev_alloc(size_t bytes);
// Returns a block from pool_dev_alloc to the cache (the caller guarantees no work
// on it is pending).
void pool_dev_free(void *p);
// Frees every cached (unused) block of every device and every cached host block;
// returns the bytes released.
size_t pool_trim();

// Host blocks (see above). host_block_free takes the size that was requested.
void *host_block_alloc(size_t bytes);
void host_block_free(void *p, size_t bytes);

// fill(dst, offset, n): produce bytes [offset, offset + n) of the source stream into
// dst (pinned staging memory).
using StageFill = std::function<void(char *dst, size_t offset, size_t n)>;
// drain(src, offset, n): consume bytes [offset, offset + n) of the device buffer from
// src (pinned staging memory).
using StageDrain = std::function<void(const char *src, size_t offset, size_t n)>;

// Host -> device copy of `bytes` produced by `fill`, on `stream`; returns after the
// last chunk has been copied (cudaError_t of the first failure).
cudaError_t staged_h2d(void *dst_dev, size_t bytes, const StageFill &fill, cudaStream_t stream);
// Device -> host copy consumed by `drain`, on `stream`; synchronous.
cudaError_t staged_d2h(const void *src_dev, size_t bytes, const StageDrain &drain, cudaStream_t stream);

// Parallel (OpenMP) memcpy used by the stage fills/drains.
void par_memcpy(void *dst, const void *src, size_t bytes);

}  // namespace topk
