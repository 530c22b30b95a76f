// host_prep.h — host-side preparation for topk_eig_create (DESIGN.md rows a1-a4):
// canonicalise (a1), symmetry check (a2), nnz-balanced partition (a3), per-part
// layout + SpMV tile table (a4). Native C++ (OpenMP where it pays).
#pragma once
#include <cstdint>
#include <memory>
#include <utility>
#include <string>
#include <vector>

#include "topk_eig.h"

namespace topk {

void *host_block_alloc(size_t bytes);  // mem_pool.cpp: cached large host blocks
void host_block_free(void *p, size_t bytes);

// Allocator that default-initialises (no zero fill) so large host buffers are
// first touched by the parallel loops that fill them; blocks of >= 1 MB come from
// the process-wide host block cache (mem_pool.h), so repeated creates reuse pages.
template <class T> struct NoInitAlloc : std::allocator<T> {
    template <class U> struct rebind { using other = NoInitAlloc<U>; };
    static constexpr size_t kBig = size_t(1) << 20;
    NoInitAlloc() = default;
    template <class U> NoInitAlloc(const NoInitAlloc<U> &) {}
    T *allocate(size_t n) {
        if (n * sizeof(T) >= kBig) return static_cast<T *>(host_block_alloc(n * sizeof(T)));
        return std::allocator<T>::allocate(n);
    }
    void deallocate(T *p, size_t n) {
        if (n * sizeof(T) >= kBig) host_block_free(p, n * sizeof(T));
        else std::allocator<T>::deallocate(p, n);
    }
    template <class U> void construct(U *p) noexcept { ::new ((void *)p) U; }
    template <class U, class... A> void construct(U *p, A &&...a) { ::new ((void *)p) U(std::forward<A>(a)...); }
};
template <class T> using hvec = std::vector<T, NoInitAlloc<T>>;

// Read-only view of a host array (borrowed from the caller's matrix, or of the
// Csr's own storage).
template <class T> struct Span {
    const T *p = nullptr;
    size_t n = 0;
    const T &operator[](size_t i) const { return p[i]; }
    const T *data() const { return p; }
    size_t size() const { return n; }
    bool empty() const { return n == 0; }
    const T &back() const { return p[n - 1]; }
};

// Canonical CSR. A CSR input that is already canonical with fp64 values is
// borrowed as is (no copy: the caller's arrays stay valid during create); any
// other input is rebuilt into the owned storage.
struct Csr {
    int64_t n = 0;
    Span<int64_t> rowptr;  // n+1
    Span<int32_t> col;     // nnz, sorted strictly increasing within each row
    Span<double> val;      // nnz
    std::vector<int64_t> rowptr_own;
    hvec<int32_t> col_own;
    hvec<double> val_own;
    void bind_owned() {
        rowptr = {rowptr_own.data(), rowptr_own.size()};
        col = {col_own.data(), col_own.size()};
        val = {val_own.data(), val_own.size()};
    }
    int64_t nnz() const { return rowptr.empty() ? 0 : rowptr.back(); }
};

// a1: COO/CSR -> canonical CSR. Duplicates summed in input order.
topk_status_t canonicalize(const topk_matrix_t &A, Csr &out, std::string &err);

// a2: structural + bitwise value symmetry (multiset hash, host_prep.cpp).
bool is_symmetric(const Csr &m);
// The four wrapping hash sums of rows [r0, r1) (upper h1, h2; transposed lower h1, h2).
// The sums are additive over row ranges, so one process per GPU checks its own rows
// and the ranks add their sums (the matrix is symmetric iff upper == lower for both).
void symmetry_sums(const Csr &m, int64_t r0, int64_t r1, uint64_t out[4]);

// a3: rule P (reading Q15). b has G+1 entries.
topk_status_t partition_rule_p(const int64_t *rowptr, int64_t n, int32_t G, int64_t *b);

// padded replica slot length: round_up(max_g n_g, 64)
int64_t padded_rows(const int64_t *b, int32_t G);

// Storage rounding (RNE, straight from f64; reading Q22).
float round_f32(double x);
uint16_t round_bf16_bits(double x);
double bf16_bits_to_double(uint16_t b);

// ---------------------------------------------------------------------------
// Local row order of a part ("degree order"): the part's
// rows sorted by (degree descending, original index ascending); empty rows
// therefore come last and the non-empty rows are positions [0, n_nonempty).
// Every part-local vector (Lanczos basis, y, w, the replica slot) is stored in
// this order; perm[p] is the original part-local row at position p.
//
// Device column entry of column c (owner part q, position p): q * n_pad + p, an
// index into the replica (= the V column at G = 1). In degree order the hub
// columns are the dense prefix of every slot, so the SpMV's plain L1-cached x
// gathers keep them resident.
// pos[r] = position of global row r inside its part's degree order.
void degree_order(const Csr &m, const int64_t *b, int32_t G, hvec<int32_t> &pos);
// colmap[c] = device column entry of global column c (one lookup per nonzero).
hvec<int32_t> column_map(int64_t n, const int64_t *b, int32_t G, int64_t npad, const int32_t *pos);

// Halo exchange (reading Q27): part g's SpMV input
// is a compact vector x_g = [own slot (n_pad) | the remote columns its rows touch,
// grouped by owner q, ascending position]; only those values cross between parts.
struct Halo {
    int64_t n = 0;               // remote entries
    std::vector<int64_t> off;    // G+1: owner q's entries are [off[q], off[q+1])
    std::vector<int32_t> pos;    // position in the owner's slot of each entry
    std::vector<int32_t> colmap; // global column -> compact device column (own: pos; remote: n_pad + t; unused: 0)
};
void build_halo(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad, const int32_t *pos, Halo &out);

// ---------------------------------------------------------------------------
// SpMV physical format (a4), derived from the logical CSR in degree order:
//  * "big" rows (positions [0, nbig), degree > kSellMaxLen) stay CSR; their
//    nonzeros are the first rowptr[nbig] entries of the physical arrays (same
//    as the logical CSR). Each big row is cut into chunks of <= kChunkNnz; a
//    warp reduces one chunk; a row with several chunks ("long row") is finished
//    by its last-arriving chunk in chunk order.
//  * the other non-empty rows form SELL-32 slices (sliced ELLPACK, C = 32,
//    sigma = the whole part): slice s = rows nbig + 32 s .. + 31, width
//    w_s = degree of its first row (rows are degree-sorted), stored column-major
//    (entry e of slice row i at base_s + 32 e + i), padded with (col = 0,
//    value 0). One lane per row, coalesced 128-byte loads, no reductions.
//  * work items: one per chunk, then groups of consecutive slices with
//    sum(w_s) <= kSellItemWidth (about <= 2048 padded nonzeros per item).
#ifndef TOPK_SELL_MAXLEN
#define TOPK_SELL_MAXLEN 128
#endif
#ifndef TOPK_CHUNK_NNZ
#define TOPK_CHUNK_NNZ 8192
#endif
#ifndef TOPK_SELL_ITEM_WIDTH
#define TOPK_SELL_ITEM_WIDTH 64
#endif
constexpr int kSellMaxLen = TOPK_SELL_MAXLEN;     // dev build variants (tools/lab/spmv_ab.py)
constexpr int kChunkNnz = TOPK_CHUNK_NNZ;
constexpr int kSellItemWidth = TOPK_SELL_ITEM_WIDTH;

struct Chunk {       // big-row chunk (24 bytes; z0 is 64-bit: parts may hold >= 2^31 nonzeros)
    int64_t z0;      // first physical nonzero
    int32_t row;     // position of the row
    int32_t cnt;     // nonzeros (<= kChunkNnz)
    int32_t long_id; // -1: the chunk is the whole row; else index into longrows
    int32_t pad;
};
struct LongRow {
    int32_t row;
    int32_t first_chunk;
    int32_t nchunks;
    int32_t pad;
};

struct PartLayout {
    int64_t row0 = 0, nrows = 0, npad = 0, nnonempty = 0;
    hvec<int64_t> rowptr;           // nrows+1, logical CSR in degree order
    hvec<int32_t> perm;             // nrows: part-local original row at each position
    // physical SpMV format
    int32_t nbig = 0;
    int64_t nphys = 0;              // physical entries (big-row CSR + padded SELL)
    hvec<int32_t> pcol;             // physical col (big-row CSR prefix, then SELL slices)
    hvec<double> pval;              // physical values
    std::vector<Chunk> chunks;
    std::vector<LongRow> longrows;
    std::vector<int64_t> sell;      // 2 per slice: base (physical index), width
    std::vector<int32_t> items;     // 2 per SELL work item: first slice, end slice
};

// Tables of one SpMV pass over a SUBSET of every row's entries (DESIGN.md section 8,
// the overlapped exchange: own-slot columns first, then the others), from the pass
// degree deg[p] of each position: big rows = positions [0, nbig) of the full layout,
// their pass entries contiguous at bigptr[p] and cut into ceil(d / kChunkNnz) chunks;
// SELL slices over [nbig, nne) with width = the largest pass degree of the slice's
// rows, padded with (col 0, value 0); slices of width 0 and big rows without pass
// entries get no work (their partial sums stay 0). With min_one = true every big row
// gets a chunk and every slice width >= 1 (the final pass finishes every non-empty
// row). With every entry in the pass this is the single-pass format above.
struct PassTables {
    std::vector<int64_t> bigptr;    // nbig+1
    std::vector<Chunk> chunks;
    std::vector<LongRow> longrows;
    std::vector<int64_t> sell;      // 2 per slice: base, width
    std::vector<int32_t> items;     // 2 per SELL work item: first slice, end slice
    int64_t nphys = 0;
};
void build_pass_tables(const int32_t *deg, int64_t nbig, int64_t nne, bool min_one, PassTables &out);

topk_status_t build_part(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad,
                         const int32_t *pos, const int32_t *colmap, PartLayout &out, std::string &err);
// The same layout without the physical arrays (perm, rowptr, chunks, long rows,
// SELL table, items, nphys): topk_eig_create scatters the nonzeros on the device
// (k_layout_big / k_layout_sell) with exactly the host rule of build_part.
topk_status_t build_part_tables(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad,
                                const int32_t *pos, PartLayout &out, std::string &err);

// The logical CSR (degree order; device column entries, values) read back out of
// the physical arrays (exports and tests).
void logical_from_physical(const PartLayout &L, hvec<int32_t> &col, hvec<double> &val);

}  // namespace topk
