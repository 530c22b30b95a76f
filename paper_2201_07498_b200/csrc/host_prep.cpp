// host_prep.cpp — rows a1-a4 of the hot-path table: canonicalise
// the input (COO as in the paper's Table I, or CSR), check
// symmetry, partition rows by nnz, and lay out each partition
// for the device (rows of M_g, replicated v_i).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include "host_prep.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace topk {

// TOPK_TRACE=1: host-preparation sub-stage times on stderr
static void hp_mark(const char *what) {
    static const bool on = [] { const char *e = std::getenv("TOPK_TRACE"); return e && e[0] == '1'; }();
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  [host_prep] %-26s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
}


static double load_value(const topk_matrix_t &A, int64_t k) {
    if (!A.values) return 1.0;
    if (A.values_dtype == TOPK_F32) return (double)((const float *)A.values)[k];
    return ((const double *)A.values)[k];
}

// Sort one row's entries by column (stable: ties keep input order) and sum
// duplicates in that order. Writes into col/val starting at `out`, returns count.
static int64_t sort_row_sum(const int32_t *cin, const double *vin, int64_t len, int32_t *cout,
                            double *vout, std::vector<int64_t> &perm) {
    bool sorted_unique = true;
    for (int64_t k = 1; k < len; ++k)
        if (cin[k] <= cin[k - 1]) { sorted_unique = false; break; }
    if (sorted_unique) {
        std::memcpy(cout, cin, (size_t)len * sizeof(int32_t));
        std::memcpy(vout, vin, (size_t)len * sizeof(double));
        return len;
    }
    perm.resize((size_t)len);
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return cin[a] < cin[b]; });
    int64_t o = 0;
    for (int64_t q = 0; q < len; ++q) {
        int64_t k = perm[(size_t)q];
        if (o > 0 && cout[o - 1] == cin[k]) {
            vout[o - 1] += vin[k];
        } else {
            cout[o] = cin[k];
            vout[o] = vin[k];
            ++o;
        }
    }
    return o;
}

topk_status_t canonicalize(const topk_matrix_t &A, Csr &out, std::string &err) {
    const int64_t n = A.n, nnz = A.nnz;
    if (n < 1 || n >= (1ll << 31) || nnz < 0) { err = "n must be in [1, 2^31) and nnz >= 0"; return TOPK_E_INVALID; }
    if (nnz > 0 && !A.col_idx) { err = "col_idx is NULL"; return TOPK_E_INVALID; }
    if (A.values && A.values_dtype != TOPK_F64 && A.values_dtype != TOPK_F32) {
        err = "values_dtype must be TOPK_F64 or TOPK_F32"; return TOPK_E_INVALID;
    }
    int bad_col = 0;
    int unsorted = 1;
    if (A.format == TOPK_CSR) {
        if (!A.row_ptr) { err = "row_ptr is NULL"; return TOPK_E_INVALID; }
        if (A.row_ptr[0] != 0 || A.row_ptr[n] != nnz) { err = "row_ptr[0] must be 0 and row_ptr[n] must be nnz"; return TOPK_E_STRUCTURE; }
        int bad_rp = 0;
#pragma omp parallel for schedule(static) reduction(| : bad_rp)
        for (int64_t r = 0; r < n; ++r) bad_rp |= (A.row_ptr[r + 1] < A.row_ptr[r]);
        if (bad_rp) { err = "row_ptr is not non-decreasing"; return TOPK_E_STRUCTURE; }
        // one pass over the entries, row by row (row_ptr is monotonic from 0 to nnz, so
        // the rows cover every entry once): range check, and whether the columns are
        // already strictly increasing in every row (canonical input -> borrowed, no copy)
        unsorted = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : bad_col, unsorted)
        for (int64_t r = 0; r < n; ++r) {
            int32_t prev = -1;
            for (int64_t k = A.row_ptr[r]; k < A.row_ptr[r + 1]; ++k) {
                const int32_t c = A.col_idx[k];
                bad_col |= (c < 0) | ((int64_t)c >= n);
                unsorted |= (c <= prev);
                prev = c;
            }
        }
    } else {
#pragma omp parallel for schedule(static) reduction(| : bad_col)
        for (int64_t k = 0; k < nnz; ++k)
            if (A.col_idx[k] < 0 || (int64_t)A.col_idx[k] >= n) bad_col = 1;
    }
    if (bad_col) { err = "column index out of range"; return TOPK_E_STRUCTURE; }
    if (A.format == TOPK_CSR) {
        if (!unsorted) {
            out.n = n;
            out.rowptr = {A.row_ptr, (size_t)n + 1};
            out.col = {A.col_idx, (size_t)nnz};
            if (A.values && A.values_dtype == TOPK_F64) {
                out.val = {static_cast<const double *>(A.values), (size_t)nnz};  // borrowed, no copy
            } else {
                out.val_own.resize((size_t)nnz);
#pragma omp parallel for schedule(static)
                for (int64_t k = 0; k < nnz; ++k) out.val_own[(size_t)k] = load_value(A, k);
                out.val = {out.val_own.data(), out.val_own.size()};
            }
            return TOPK_OK;
        }
    }

    // Gather entries grouped by row, preserving input order inside a row.
    std::vector<int64_t> start((size_t)n + 1, 0);
    hvec<int32_t> gcol((size_t)nnz);
    hvec<double> gval((size_t)nnz);
    if (A.format == TOPK_CSR) {
        if (!A.row_ptr) { err = "row_ptr is NULL"; return TOPK_E_INVALID; }
        if (A.row_ptr[0] != 0 || A.row_ptr[n] != nnz) { err = "row_ptr[0] must be 0 and row_ptr[n] must be nnz"; return TOPK_E_STRUCTURE; }
        for (int64_t r = 0; r < n; ++r)
            if (A.row_ptr[r + 1] < A.row_ptr[r]) { err = "row_ptr is not non-decreasing"; return TOPK_E_STRUCTURE; }
        std::memcpy(start.data(), A.row_ptr, (size_t)(n + 1) * sizeof(int64_t));
        std::memcpy(gcol.data(), A.col_idx, (size_t)nnz * sizeof(int32_t));
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < nnz; ++k) gval[(size_t)k] = load_value(A, k);
    } else if (A.format == TOPK_COO) {
        if (nnz > 0 && !A.row_idx) { err = "row_idx is NULL"; return TOPK_E_INVALID; }
        for (int64_t k = 0; k < nnz; ++k)
            if (A.row_idx[k] < 0 || A.row_idx[k] >= n) { err = "row index out of range"; return TOPK_E_STRUCTURE; }
        for (int64_t k = 0; k < nnz; ++k) start[(size_t)A.row_idx[k] + 1]++;
        std::partial_sum(start.begin(), start.end(), start.begin());
        std::vector<int64_t> pos(start.begin(), start.end() - 1);
        for (int64_t k = 0; k < nnz; ++k) {
            int64_t p = pos[(size_t)A.row_idx[k]]++;
            gcol[(size_t)p] = A.col_idx[k];
            gval[(size_t)p] = load_value(A, k);
        }
    } else {
        err = "unknown matrix format"; return TOPK_E_INVALID;
    }

    // Per row: stable sort by column, sum duplicates; then compact.
    std::vector<int64_t> cnt((size_t)n, 0);
    out.n = n;
    out.col_own.resize((size_t)nnz);
    out.val_own.resize((size_t)nnz);
#pragma omp parallel
    {
        std::vector<int64_t> perm;
#pragma omp for schedule(dynamic, 1024)
        for (int64_t r = 0; r < n; ++r) {
            int64_t b = start[(size_t)r], len = start[(size_t)r + 1] - b;
            cnt[(size_t)r] = sort_row_sum(gcol.data() + b, gval.data() + b, len,
                                          out.col_own.data() + b, out.val_own.data() + b, perm);
        }
    }
    out.rowptr_own.assign((size_t)n + 1, 0);
    for (int64_t r = 0; r < n; ++r) out.rowptr_own[(size_t)r + 1] = out.rowptr_own[(size_t)r] + cnt[(size_t)r];
    if (out.rowptr_own[(size_t)n] != nnz) {  // duplicates were merged: compact in place
        for (int64_t r = 0; r < n; ++r) {
            int64_t src = start[(size_t)r], dst = out.rowptr_own[(size_t)r];
            if (src != dst) {
                std::memmove(out.col_own.data() + dst, out.col_own.data() + src, (size_t)cnt[(size_t)r] * sizeof(int32_t));
                std::memmove(out.val_own.data() + dst, out.val_own.data() + src, (size_t)cnt[(size_t)r] * sizeof(double));
            }
        }
        out.col_own.resize((size_t)out.rowptr_own[(size_t)n]);
        out.val_own.resize((size_t)out.rowptr_own[(size_t)n]);
    }
    out.bind_owned();
    return TOPK_OK;
}

// a2 (reading Q17): M = M^T structurally and bitwise in values. The canonical CSR has
// no duplicates, so this holds iff the multiset of off-diagonal entries (r, c, bits)
// with c > r equals the multiset of (c, r, bits) with c < r. Both multisets are
// compared through two independent 64-bit hash sums (wrapping addition) of the entry
// key (min(r,c) << 32 | max(r,c), unique because n < 2^31) and the value bits: a
// symmetric matrix always passes; an asymmetric one passes only on a simultaneous
// collision of both sums (probability ~2^-128 for random-function hashes). One
// parallel pass over the nonzeros (a binary search per nonzero took 1.8 s at C3).
// Two finalisers per entry: splitmix64's and murmur3's fmix64 (different constants).
static inline uint64_t sym_mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static inline uint64_t sym_fmix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    return x ^ (x >> 33);
}
bool is_symmetric(const Csr &m) {
    uint64_t h[4];
    symmetry_sums(m, 0, m.n, h);
    return h[0] == h[2] && h[1] == h[3];
}

void symmetry_sums(const Csr &m, int64_t r0, int64_t r1, uint64_t out[4]) {
    uint64_t u1 = 0, u2 = 0, l1 = 0, l2 = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : u1, u2, l1, l2)
    for (int64_t r = r0; r < r1; ++r) {
        for (int64_t k = m.rowptr[(size_t)r]; k < m.rowptr[(size_t)r + 1]; ++k) {
            const int64_t c = m.col[(size_t)k];
            if (c == r) continue;
            uint64_t vb;
            const double v = m.val[(size_t)k];
            std::memcpy(&vb, &v, 8);
            const uint64_t key = ((uint64_t)std::min(r, c) << 32) | (uint64_t)std::max(r, c);
            const uint64_t h1 = sym_mix(key ^ (vb * 0x9E3779B97F4A7C15ull));
            const uint64_t h2 = sym_fmix((key * 0xD6E8FEB86659FD93ull) ^ (vb + 0x2545F4914F6CDD1Dull));
            if (c > r) { u1 += h1; u2 += h2; } else { l1 += h1; l2 += h2; }
        }
    }
    out[0] = u1; out[1] = u2; out[2] = l1; out[3] = l2;
}

// Number of parts a left-to-right greedy packing with bottleneck B needs,
// jumping part by part with binary searches on the prefix sum rowptr.
static int64_t parts_needed(const int64_t *rowptr, int64_t n, int64_t B, int64_t cap) {
    int64_t s = 0, parts = 0;
    while (s < n) {
        ++parts;
        if (parts > cap) return parts;
        // last row index e (exclusive) with rowptr[e] - rowptr[s] <= B
        const int64_t *p = std::upper_bound(rowptr + s, rowptr + n + 1, rowptr[s] + B);
        int64_t e = (int64_t)(p - rowptr) - 1;
        if (e <= s) return INT64_MAX;  // a single row exceeds B
        s = e;
    }
    return parts;
}

topk_status_t partition_rule_p(const int64_t *rowptr, int64_t n, int32_t G, int64_t *b) {
    if (G < 1 || n < G) return TOPK_E_INVALID;
    int64_t maxrow = 0;
#pragma omp parallel for schedule(static) reduction(max : maxrow)
    for (int64_t r = 0; r < n; ++r) maxrow = std::max(maxrow, rowptr[r + 1] - rowptr[r]);
    int64_t lo = maxrow, hi = std::max(maxrow, rowptr[n]);
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (parts_needed(rowptr, n, mid, G) <= G) hi = mid; else lo = mid + 1;
    }
    const int64_t Bs = lo;
    b[G] = n;
    for (int32_t k = G - 1; k >= 1; --k) {
        int64_t target = rowptr[b[k + 1]] - Bs;
        int64_t j = (int64_t)(std::lower_bound(rowptr, rowptr + n + 1, target) - rowptr);
        b[k] = std::max<int64_t>(j, k);
    }
    b[0] = 0;
    return TOPK_OK;
}

int64_t padded_rows(const int64_t *b, int32_t G) {
    int64_t mx = 0;
    for (int32_t g = 0; g < G; ++g) mx = std::max(mx, b[g + 1] - b[g]);
    return (mx + 63) / 64 * 64;
}

float round_f32(double x) { return (float)x; }

uint16_t round_bf16_bits(double x) {
    // f64 -> f32 with round-to-odd, then f32 -> bf16 round-to-nearest-even:
    // exact single rounding because f32 keeps 16 more bits than bf16.
    float f = (float)x;
    if (std::isfinite(x) && (double)f != x) {
        if (std::fabs((double)f) > std::fabs(x)) f = std::nextafter(f, 0.0f);
        uint32_t fb;
        std::memcpy(&fb, &f, 4);
        fb |= 1u;
        std::memcpy(&f, &fb, 4);
    }
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

double bf16_bits_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return (double)f;
}



// a[i] <- a[0] + ... + a[i] (parallel: per-thread chunk sums, a serial scan over the
// threads' totals, then each chunk offset; identical to the serial running sum)
static void prefix_sum_inplace(int64_t *a, int64_t n) {
    const int T = n >= (1 << 20) ? std::max(1, omp_get_max_threads()) : 1;
    if (T == 1) {
        for (int64_t i = 1; i < n; ++i) a[i] += a[i - 1];
        return;
    }
    std::vector<int64_t> tot((size_t)T + 1, 0);
    const int64_t per = (n + T - 1) / T;
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int t = 0; t < T; ++t) {
        const int64_t i0 = std::min(n, (int64_t)t * per), i1 = std::min(n, i0 + per);
        int64_t run = 0;
        for (int64_t i = i0; i < i1; ++i) { run += a[i]; a[i] = run; }
        tot[(size_t)t + 1] = run;
    }
    for (int t = 0; t < T; ++t) tot[(size_t)t + 1] += tot[(size_t)t];
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int t = 0; t < T; ++t) {
        const int64_t i0 = std::min(n, (int64_t)t * per), i1 = std::min(n, i0 + per);
        const int64_t off = tot[(size_t)t];
        if (off)
            for (int64_t i = i0; i < i1; ++i) a[i] += off;
    }
}

void degree_order(const Csr &m, const int64_t *b, int32_t G, hvec<int32_t> &pos) {
    // stable counting sort by degree, descending (ties keep ascending row index)
    pos.resize((size_t)m.n);
    auto deg = [&](int64_t r) { return m.rowptr[(size_t)r + 1] - m.rowptr[(size_t)r]; };
    for (int32_t q = 0; q < G; ++q) {
        const int64_t a = b[q], e = b[q + 1], nr = e - a;
        int64_t dmax = 0;
#pragma omp parallel for schedule(static) reduction(max : dmax)
        for (int64_t r = a; r < e; ++r) dmax = std::max(dmax, deg(r));
        const int64_t nb = dmax + 1;  // key = dmax - degree
        const int T = (nr >= (1 << 16) && nb <= (1 << 22)) ? std::max(1, omp_get_max_threads()) : 1;
        // per-thread histograms over contiguous row chunks; positions = (key, thread, row) order
        hvec<int64_t> cnt((size_t)T * (size_t)nb);
        const int64_t per = (nr + T - 1) / T;
#pragma omp parallel for schedule(static, 1) num_threads(T)
        for (int t = 0; t < T; ++t) std::fill(cnt.data() + (size_t)t * nb, cnt.data() + (size_t)(t + 1) * nb, int64_t(0));
#pragma omp parallel for schedule(static, 1) num_threads(T)
        for (int t = 0; t < T; ++t) {
            int64_t *c = cnt.data() + (size_t)t * nb;
            const int64_t r1 = std::min(e, a + (t + 1) * per);
            for (int64_t r = a + t * per; r < r1; ++r) c[dmax - deg(r)]++;
        }
        int64_t run = 0;
        for (int64_t k = 0; k < nb; ++k)
            for (int t = 0; t < T; ++t) {
                int64_t &c = cnt[(size_t)t * nb + (size_t)k];
                const int64_t v = c;
                c = run;
                run += v;
            }
#pragma omp parallel for schedule(static, 1) num_threads(T)
        for (int t = 0; t < T; ++t) {
            int64_t *c = cnt.data() + (size_t)t * nb;
            const int64_t r1 = std::min(e, a + (t + 1) * per);
            for (int64_t r = a + t * per; r < r1; ++r) pos[(size_t)r] = (int32_t)c[dmax - deg(r)]++;
        }
    }
}


hvec<int32_t> column_map(int64_t n, const int64_t *b, int32_t G, int64_t npad, const int32_t *pos) {
    hvec<int32_t> cm((size_t)n);
    for (int32_t q = 0; q < G; ++q) {
#pragma omp parallel for schedule(static)
        for (int64_t c = b[q]; c < b[q + 1]; ++c) cm[(size_t)c] = (int32_t)(q * npad + pos[(size_t)c]);
    }
    return cm;
}

void build_halo(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad, const int32_t *pos, Halo &out) {
    const int64_t n = m.n;
    const int64_t z0 = m.rowptr[(size_t)b[g]], z1 = m.rowptr[(size_t)b[g + 1]];
    // columns touched by part g's rows (benign same-value races)
    std::vector<uint8_t> used((size_t)n, 0);
#pragma omp parallel for schedule(static)
    for (int64_t k = z0; k < z1; ++k) used[(size_t)m.col[(size_t)k]] = 1;
    out.colmap.assign((size_t)n, 0);
    out.off.assign((size_t)G + 1, 0);
    out.pos.clear();
    for (int32_t q = 0; q < G; ++q) {
        const int64_t a = b[q], e = b[q + 1];
        if (q == g) {
#pragma omp parallel for schedule(static)
            for (int64_t c = a; c < e; ++c) out.colmap[(size_t)c] = pos[(size_t)c];
            out.off[(size_t)q + 1] = out.off[(size_t)q];
            continue;
        }
        // marked owner positions in ascending order: position-indexed flags, then a scan
        std::vector<int32_t> row_at((size_t)(e - a), -1);
        for (int64_t c = a; c < e; ++c)
            if (used[(size_t)c]) row_at[(size_t)pos[(size_t)c]] = (int32_t)(c - a);
        const int64_t base = out.off[(size_t)q];
        int64_t t = 0;
        for (int64_t p = 0; p < e - a; ++p) {
            const int32_t rr = row_at[(size_t)p];
            if (rr < 0) continue;
            out.pos.push_back((int32_t)p);
            out.colmap[(size_t)(a + rr)] = (int32_t)(npad + base + t);
            ++t;
        }
        out.off[(size_t)q + 1] = base + t;
    }
    out.n = out.off[(size_t)G];
}

topk_status_t build_part_tables(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad,
                                const int32_t *pos, PartLayout &out, std::string &err) {
    const int64_t r0 = b[g], r1 = b[g + 1];
    const int64_t z0 = m.rowptr[(size_t)r0], z1 = m.rowptr[(size_t)r1];
    hp_mark("build_part: start");
    (void)z0; (void)z1;  // any per-part nnz (64-bit offsets)
    if ((int64_t)G * npad >= (1ll << 31)) { err = "G * n_pad must be < 2^31"; return TOPK_E_INVALID; }
    (void)G;
    out.row0 = r0;
    out.nrows = r1 - r0;
    out.npad = npad;
    const int64_t ng = r1 - r0;
    out.perm.resize((size_t)ng);
#pragma omp parallel for schedule(static)
    for (int64_t r = r0; r < r1; ++r) out.perm[(size_t)pos[(size_t)r]] = (int32_t)(r - r0);
    out.rowptr.resize((size_t)(ng + 1));
    out.rowptr[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < ng; ++p) {  // row lengths in degree order (random reads, parallel)
        const int64_t r = r0 + out.perm[(size_t)p];
        out.rowptr[(size_t)p + 1] = m.rowptr[(size_t)r + 1] - m.rowptr[(size_t)r];
    }
    // lengths are non-increasing in degree order: the non-empty rows are a prefix
    int64_t nne = 0;
#pragma omp parallel for schedule(static) reduction(max : nne)
    for (int64_t p = 0; p < ng; ++p)
        if (out.rowptr[(size_t)p + 1] > 0) nne = std::max(nne, p + 1);
    out.nnonempty = nne;
    prefix_sum_inplace(out.rowptr.data() + 1, ng);
    hp_mark("perm + rowptr");
    // physical format: big rows (CSR prefix, chunked), then SELL-32 slices
    int64_t nbig = 0;
    while (nbig < nne && out.rowptr[(size_t)nbig + 1] - out.rowptr[(size_t)nbig] > kSellMaxLen) ++nbig;
    out.nbig = (int32_t)nbig;
    out.chunks.clear();
    out.longrows.clear();
    for (int64_t p = 0; p < nbig; ++p) {
        const int64_t rb = out.rowptr[(size_t)p], len = out.rowptr[(size_t)p + 1] - rb;
        const int32_t nch = (int32_t)((len + kChunkNnz - 1) / kChunkNnz);
        const int32_t lid = nch > 1 ? (int32_t)out.longrows.size() : -1;
        if (nch > 1) out.longrows.push_back(LongRow{(int32_t)p, (int32_t)out.chunks.size(), nch, 0});
        for (int32_t c = 0; c < nch; ++c)
            out.chunks.push_back(Chunk{rb + (int64_t)c * kChunkNnz, (int32_t)p,
                                       (int32_t)std::min<int64_t>(kChunkNnz, len - (int64_t)c * kChunkNnz), lid, 0});
    }
    const int64_t zbig = out.rowptr[(size_t)nbig];
    const int64_t nsl = (nne - nbig + 31) / 32;
    out.sell.assign((size_t)(2 * nsl), 0);
    // slice widths in parallel, bases = zbig + 32 * (exclusive prefix of the widths)
    hvec<int64_t> span((size_t)nsl);
#pragma omp parallel for schedule(static)
    for (int64_t sl = 0; sl < nsl; ++sl) {
        const int64_t p0 = nbig + 32 * sl;
        span[(size_t)sl] = 32 * (out.rowptr[(size_t)p0 + 1] - out.rowptr[(size_t)p0]);
    }
    prefix_sum_inplace(span.data(), nsl);
#pragma omp parallel for schedule(static)
    for (int64_t sl = 0; sl < nsl; ++sl) {
        const int64_t incl = span[(size_t)sl], prev = sl ? span[(size_t)sl - 1] : 0;
        out.sell[(size_t)(2 * sl)] = zbig + prev;
        out.sell[(size_t)(2 * sl + 1)] = (incl - prev) / 32;
    }
    const int64_t phys = zbig + (nsl ? span[(size_t)nsl - 1] : 0);
    out.items.clear();
    for (int64_t sl = 0; sl < nsl;) {
        int64_t e = sl, width = 0;
        while (e < nsl && (e == sl || width + out.sell[(size_t)(2 * e + 1)] <= kSellItemWidth)) {
            width += out.sell[(size_t)(2 * e + 1)];
            ++e;
        }
        out.items.push_back((int32_t)sl);
        out.items.push_back((int32_t)e);
        sl = e;
    }
    out.nphys = phys;
    hp_mark("chunks + slices + items");
    return TOPK_OK;
}

void build_pass_tables(const int32_t *deg, int64_t nbig, int64_t nne, bool min_one, PassTables &out) {
    out.bigptr.assign((size_t)nbig + 1, 0);
    for (int64_t p = 0; p < nbig; ++p) out.bigptr[(size_t)p + 1] = out.bigptr[(size_t)p] + deg[(size_t)p];
    out.chunks.clear();
    out.longrows.clear();
    for (int64_t p = 0; p < nbig; ++p) {
        const int64_t rb = out.bigptr[(size_t)p], len = out.bigptr[(size_t)p + 1] - rb;
        int32_t nch = (int32_t)((len + kChunkNnz - 1) / kChunkNnz);
        if (nch == 0 && min_one) nch = 1;
        const int32_t lid = nch > 1 ? (int32_t)out.longrows.size() : -1;
        if (nch > 1) out.longrows.push_back(LongRow{(int32_t)p, (int32_t)out.chunks.size(), nch, 0});
        for (int32_t c = 0; c < nch; ++c)
            out.chunks.push_back(Chunk{rb + (int64_t)c * kChunkNnz, (int32_t)p,
                                       (int32_t)std::max<int64_t>(0, std::min<int64_t>(kChunkNnz, len - (int64_t)c * kChunkNnz)),
                                       lid, 0});
    }
    const int64_t nsl = (nne - nbig + 31) / 32;
    out.sell.assign((size_t)(2 * nsl), 0);
#pragma omp parallel for schedule(static)
    for (int64_t sl = 0; sl < nsl; ++sl) {
        const int64_t p0 = nbig + 32 * sl, p1 = std::min(nne, p0 + 32);
        int64_t w = min_one ? 1 : 0;
        for (int64_t p = p0; p < p1; ++p) w = std::max<int64_t>(w, deg[(size_t)p]);
        out.sell[(size_t)(2 * sl + 1)] = w;
    }
    int64_t phys = out.bigptr[(size_t)nbig];
    for (int64_t sl = 0; sl < nsl; ++sl) {
        out.sell[(size_t)(2 * sl)] = phys;
        phys += 32 * out.sell[(size_t)(2 * sl + 1)];
    }
    out.items.clear();
    for (int64_t sl = 0; sl < nsl;) {
        if (out.sell[(size_t)(2 * sl + 1)] == 0) { ++sl; continue; }  // nothing of this pass in the slice
        int64_t e = sl, width = 0;
        while (e < nsl && out.sell[(size_t)(2 * e + 1)] > 0 &&
               (e == sl || width + out.sell[(size_t)(2 * e + 1)] <= kSellItemWidth)) {
            width += out.sell[(size_t)(2 * e + 1)];
            ++e;
        }
        out.items.push_back((int32_t)sl);
        out.items.push_back((int32_t)e);
        sl = e;
    }
    out.nphys = phys;
}

topk_status_t build_part(const Csr &m, const int64_t *b, int32_t G, int32_t g, int64_t npad,
                         const int32_t *pos, const int32_t *colmap, PartLayout &out, std::string &err) {
    topk_status_t s = build_part_tables(m, b, G, g, npad, pos, out, err);
    if (s != TOPK_OK) return s;
    const int64_t r0 = b[g];
    const int64_t nne = out.nnonempty, nbig = out.nbig, phys = out.nphys;
    const int64_t nsl = (int64_t)out.sell.size() / 2;
    out.pcol.resize((size_t)phys);
    out.pval.resize((size_t)phys);
    // every entry straight from the canonical CSR to its physical slot (rows in
    // degree order, entries of a row in their column-sorted input order)
#pragma omp parallel for schedule(dynamic, 2048)
    for (int64_t p = 0; p < nne; ++p) {
        const int64_t r = r0 + out.perm[(size_t)p];
        const int64_t kb = m.rowptr[(size_t)r], len = m.rowptr[(size_t)r + 1] - kb;
        size_t dst, stride;
        if (p < nbig) {
            dst = (size_t)out.rowptr[(size_t)p];
            stride = 1;
        } else {
            const int64_t sl = (p - nbig) / 32, i = (p - nbig) % 32;
            dst = (size_t)(out.sell[(size_t)(2 * sl)] + i);
            stride = 32;
        }
        for (int64_t e = 0; e < len; ++e, dst += stride) {
            out.pcol[dst] = colmap[(size_t)m.col[(size_t)(kb + e)]];
            out.pval[dst] = m.val[(size_t)(kb + e)];
        }
    }
    hp_mark("scatter");
    // SELL padding: (column 0, value 0) past each row's length
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t sl = 0; sl < nsl; ++sl) {
        const int64_t base = out.sell[(size_t)(2 * sl)], w = out.sell[(size_t)(2 * sl + 1)];
        for (int64_t i = 0; i < 32; ++i) {
            const int64_t p = nbig + 32 * sl + i;
            const int64_t len = p < nne ? out.rowptr[(size_t)p + 1] - out.rowptr[(size_t)p] : 0;
            for (int64_t e = len; e < w; ++e) {
                out.pcol[(size_t)(base + 32 * e + i)] = 0;
                out.pval[(size_t)(base + 32 * e + i)] = 0.0;
            }
        }
    }
    hp_mark("padding");
    return TOPK_OK;
}

void logical_from_physical(const PartLayout &L, hvec<int32_t> &col, hvec<double> &val) {
    const int64_t z = L.rowptr.empty() ? 0 : L.rowptr.back();
    col.resize((size_t)z);
    val.resize((size_t)z);
    for (int64_t p = 0; p < L.nnonempty; ++p) {
        const int64_t rb = L.rowptr[(size_t)p], len = L.rowptr[(size_t)p + 1] - rb;
        for (int64_t e = 0; e < len; ++e) {
            size_t src;
            if (p < L.nbig) src = (size_t)(rb + e);
            else {
                const int64_t sl = (p - L.nbig) / 32, i = (p - L.nbig) % 32;
                src = (size_t)(L.sell[(size_t)(2 * sl)] + 32 * e + i);
            }
            col[(size_t)(rb + e)] = L.pcol[src];
            val[(size_t)(rb + e)] = L.pval[src];
        }
    }
}

}  // namespace topk
