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

// Allocator that default-initialises (no zero fill) so large host buffers are
// first touched by the parallel loops that fill them.
template <class T> struct NoInitAlloc : std::allocator<T> {
    template <class U> struct rebind { using other = NoInitAlloc<U>; };
    NoInitAlloc() = default;
    template <class U> NoInitAlloc(const NoInitAlloc<U> &) {}
    template <class U> void construct(U *p) noexcept { ::new ((void *)p) U; }
    template <class U, class... A> void construct(U *p, A &&...a) { ::new ((void *)p) U(std::forward<A>(a)...); }
};
template <class T> using hvec = std::vector<T, NoInitAlloc<T>>;

struct Csr {
    int64_t n = 0;
    std::vector<int64_t> rowptr;  // n+1
    hvec<int32_t> col;            // nnz, sorted strictly increasing within each row
    hvec<double> val;             // nnz
    int64_t nnz() const { return rowptr.empty() ? 0 : rowptr.back(); }
};

// a1: COO/CSR -> canonical CSR. Duplicates summed in input order.
topk_status_t canonicalize(const topk_matrix_t &A, Csr &out, std::string &err);

// a2: structural + bitwise value symmetry.
bool is_symmetric(const Csr &m);

// a3: rule P (reading Q15). b has G+1 entries.
topk_status_t partition_rule_p(const int64_t *rowptr, int64_t n, int32_t G, int64_t *b);

// padded replica slot length: round_up(max_g n_g, 64)
int64_t padded_rows(const int64_t *b, int32_t G);

// Storage rounding (RNE, straight from f64; reading Q22).
float round_f32(double x);
uint16_t round_bf16_bits(double x);
double bf16_bits_to_double(uint16_t b);

// SpMV tile table (a4). A packed tile covers consecutive NON-EMPTY rows whose
// nonzeros total <= kTileNnz (whole rows only); a row with more than kTileNnz
// nonzeros is split into fixed kTileNnz chunks ("long row"). Empty rows belong
// to no tile: their SpMV output is identically 0 (y is zeroed once at create).
// Row ends are a bitmask over the part's nonzeros (bit k set iff k is the last
// nonzero of its row). In the hub-first order the non-empty rows are positions
// [0, n_nonempty), so the j-th row end of a tile is row end_begin + j and the
// kernel never reads rowptr.
constexpr int kTileNnz = 1024;

struct Tile {
    int32_t nz_begin;   // first nonzero (part-local) of the tile / chunk
    int32_t cnt;        // nonzeros in the tile / chunk (<= kTileNnz)
    int32_t end_begin;  // position (= index among non-empty rows) of the tile's first row
    int32_t long_id;    // -1 packed; else index into the long-row table
};
struct LongRow {
    int32_t row;
    int32_t first_tile;
    int32_t nchunks;
    int32_t pad;
};

struct PartLayout {
    int64_t row0 = 0, nrows = 0, npad = 0;
    std::vector<int32_t> rowptr;    // nrows+1, rebased
    hvec<int32_t> col;              // remapped into the padded replica index space
    hvec<double> val;               // values (f64 source; rounded to the value dtype at upload)
    std::vector<Tile> tiles;
    std::vector<LongRow> longrows;
    std::vector<uint32_t> endbits;  // ceil(nnz / 32) + 1 words
    std::vector<int32_t> nzrow;     // positions of the non-empty rows, ascending
    std::vector<int32_t> perm;      // nrows: part-local original row at each position
};

// Hot rows/columns: the H non-empty rows of largest degree
// (row nnz = column nnz, M symmetric), ties by lower index, H = kHotBytes /
// (vector storage bytes) so their x values fill ~192 KB of L1. Their col entries
// carry bit 31 so the SpMV gathers them evict-last into L1 while all other
// gathers bypass L1 allocation. Local row order of a part ("hub-first"): hot rows
// (degree descending, index ascending), then the other non-empty rows ascending,
// then the empty rows ascending -- so the hot x values are packed densely in
// 32-byte sectors and the non-empty rows are exactly positions [0, n_nonempty).
constexpr int64_t kHotBytes = 192 * 1024;
constexpr uint32_t kHotBit = 0x80000000u;
int64_t hot_count(int64_t n, int storage_bytes);
std::vector<uint8_t> hot_columns(const Csr &m, int64_t H);
// pos[r] = position of global row r inside its part's hub-first order;
// perm_g[p] = part-local original row at position p.
void hub_first_order(const Csr &m, const int64_t *b, int32_t G, const uint8_t *hot,
                     std::vector<int32_t> &pos);

// colmap[c] = owner(c) * npad + pos[c], | kHotBit if c is hot: the device column
// index of global column c (one lookup per nonzero in build_part).
std::vector<int32_t> column_map(int64_t n, const int64_t *b, int32_t G, int64_t npad, const uint8_t *hot,
                                const int32_t *pos);

topk_status_t build_part(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad,
                         const int32_t *pos, const int32_t *colmap, PartLayout &out, std::string &err);

}  // namespace topk
