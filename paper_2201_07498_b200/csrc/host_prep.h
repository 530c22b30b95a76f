// host_prep.h — host-side preparation for topk_eig_create (DESIGN.md rows a1-a4):
// canonicalise (a1), symmetry check (a2), nnz-balanced partition (a3), per-part
// layout + SpMV tile table (a4). Native C++ (OpenMP where it pays).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "topk_eig.h"

namespace topk {

struct Csr {
    int64_t n = 0;
    std::vector<int64_t> rowptr;  // n+1
    std::vector<int32_t> col;     // nnz, sorted strictly increasing within each row
    std::vector<double> val;      // nnz
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

// SpMV tile table (a4). A packed tile covers whole rows [row_begin, row_end)
// with at most kTileNnz nonzeros and kTileRows rows; a row with more than
// kTileNnz nonzeros is split into fixed chunks ("long row").
constexpr int kTileNnz = 2048;
constexpr int kTileRows = 2048;

struct Tile {
    int32_t row_begin;
    int32_t row_end;
    int32_t nz_begin;  // first nonzero (part-local) of the tile
    int32_t long_id;   // -1 packed; else index into the long-row table
};
struct LongRow {
    int32_t row;
    int32_t first_tile;
    int32_t nchunks;
    int32_t pad;
};

struct PartLayout {
    int64_t row0 = 0, nrows = 0, npad = 0;
    std::vector<int32_t> rowptr;  // nrows+1, rebased
    std::vector<int32_t> col;     // remapped into the padded replica index space
    std::vector<double> val;      // values (f64 source; rounded to the value dtype at upload)
    std::vector<Tile> tiles;
    std::vector<LongRow> longrows;
};

topk_status_t build_part(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad,
                         PartLayout &out, std::string &err);

}  // namespace topk
