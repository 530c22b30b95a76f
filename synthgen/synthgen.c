/*
 * synthgen.c — seeded synthetic INPUT generators (ER, R-MAT, Dirichlet path,
 * path/cycle Laplacians, 2-D grids).
 *
 * This module is input infrastructure shared by the oracle (oracle/) and the
 * CUDA path (paper_2201_07498_b200/). It holds none of the eigensolver's
 * arithmetic: it only produces matrices whose shape mimics the paper's
 * workloads (Table I: SuiteSparse graphs; GAP-kron is a
 * Graph500 R-MAT) and the closed-form test matrices of BASELINE.json config 2.
 * Recipes are stated in DESIGN.md ("Input recipe") and SURVEY.md 8(d).
 *
 * Randomness: a counter-based hash (splitmix64 finaliser), so every sample is
 * a pure function of (seed, sample index, draw index) and the generators are
 * deterministic regardless of OpenMP thread count.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n;
    int64_t nnz;
    int64_t *rowptr; /* n+1 */
    int32_t *col;    /* nnz */
    double *val;     /* nnz */
} sg_csr_t;

static inline uint64_t sg_mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
static inline uint64_t sg_h3(uint64_t s, uint64_t a, uint64_t b) {
    return sg_mix(sg_mix(sg_mix(s) ^ a) ^ b);
}
static inline double sg_unit(uint64_t x) { /* U[0,1) with 53 random bits */
    return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

uint64_t sg_hash3(uint64_t s, uint64_t a, uint64_t b) { return sg_h3(s, a, b); }

void sg_free(sg_csr_t *m) {
    if (!m) return;
    free(m->rowptr);
    free(m->col);
    free(m->val);
    free(m);
}

/* LSD radix sort of n 64-bit keys on their low key_bits bits (11-bit digits), with a
 * caller-provided scratch of n keys; the result is in keys. Used to build CSR. */
static int radix_sort_u64_buf(uint64_t *keys, uint64_t *tmp, int64_t n, int key_bits) {
    int64_t *cnt = (int64_t *)malloc(2048 * sizeof(int64_t));
    if (!cnt) return -1;
    uint64_t *src = keys, *dst = tmp;
    for (int shift = 0; shift < key_bits; shift += 11) {
        memset(cnt, 0, 2048 * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) cnt[(src[i] >> shift) & 0x7FF]++;
        int64_t s = 0;
        for (int d = 0; d < 2048; ++d) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
        for (int64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & 0x7FF]++] = src[i];
        uint64_t *t = src; src = dst; dst = t;
    }
    if (src != keys) memcpy(keys, src, (size_t)n * sizeof(uint64_t));
    free(cnt);
    return 0;
}

/* ------------------------------------------------------------------ */
/* R-MAT (Graph500 recursive matrix) symmetric graph.
 *   sample e, level l: r = U(h3(seed, e, l)) picks a quadrant with
 *   probabilities (a, b, c, 1-a-b-c); MSB first. Vertex ids are scrambled by a
 *   seeded bijection on [0, 2^S) (3 rounds of x <- (A_r x + C_r) mod 2^S,
 *   x ^= x >> 11). Ids >= n are rejected; self loops dropped; both directions
 *   emitted; duplicates removed. Weight of edge {u,v} = k/128 with
 *   k = 64 + (h3(seed ^ W, min, max) >> 57) in [64,191]: exactly representable
 *   in bf16, f32 and f64, so the matrix is identical in every storage mode. */
static inline uint64_t rmat_scramble(uint64_t x, int S, const uint64_t *A, const uint64_t *C) {
    uint64_t mask = (S >= 64) ? ~0ull : ((1ull << S) - 1);
    for (int r = 0; r < 3; ++r) {
        x = (A[r] * x + C[r]) & mask;
        x ^= x >> 11;
    }
    return x;
}

sg_csr_t *sg_rmat(int scale, int64_t n, int64_t samples, double a, double b, double c,
                  uint64_t seed) {
    if (scale < 1 || scale > 30 || n < 1 || n > (1ll << scale) || samples < 0) return NULL;
    uint64_t A[3], C[3];
    uint64_t mask = (1ull << scale) - 1;
    for (int r = 0; r < 3; ++r) {
        A[r] = (sg_mix(seed ^ (0xA5A5A5A5ull * (uint64_t)(r + 1))) | 1ull) & mask;
        C[r] = sg_mix(seed ^ (0x3C3C3C3C5Aull * (uint64_t)(r + 1))) & mask;
        if (A[r] == 0) A[r] = 1;
    }
    uint64_t *keys = (uint64_t *)malloc((size_t)(2 * samples + 1) * sizeof(uint64_t));
    if (!keys) return NULL;
    const double ab = a + b, abc = a + b + c;
    /* two-pass deterministic fill: every sample writes slots 2e, 2e+1; rejected
       samples write a sentinel that is squeezed out afterwards. */
    const uint64_t SENT = ~0ull;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < samples; ++e) {
        uint64_t u = 0, v = 0;
        for (int l = 0; l < scale; ++l) {
            double r = sg_unit(sg_h3(seed, (uint64_t)e, (uint64_t)l));
            uint64_t bu, bv;
            if (r < a) { bu = 0; bv = 0; }
            else if (r < ab) { bu = 0; bv = 1; }
            else if (r < abc) { bu = 1; bv = 0; }
            else { bu = 1; bv = 1; }
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        u = rmat_scramble(u, scale, A, C);
        v = rmat_scramble(v, scale, A, C);
        if (u == v || (int64_t)u >= n || (int64_t)v >= n) {
            keys[2 * e] = SENT;
            keys[2 * e + 1] = SENT;
        } else {
            keys[2 * e] = (u << scale) | v;
            keys[2 * e + 1] = (v << scale) | u;
        }
    }
    /* sort + dedupe in parallel (identical output to a serial sort of all keys):
       scatter the non-sentinel keys into 2^B buckets by their top B bits (each bucket
       = a disjoint row range), LSD-radix-sort every bucket, drop duplicates, build
       the CSR rows of each bucket independently */
    const int kb = 2 * scale;
    const int B = scale < 12 ? scale : 12;
    const int64_t NB = (int64_t)1 << B;
    const int low = kb - B;  /* bits below the bucket id */
    const int64_t ntot = 2 * samples;
    uint64_t *tmp = (uint64_t *)malloc((size_t)(ntot + 1) * sizeof(uint64_t));
    int nth = 1;
#ifdef _OPENMP
    nth = omp_get_max_threads();
#endif
    int64_t *hist = (int64_t *)calloc((size_t)nth * NB, sizeof(int64_t));
    int64_t *boff = (int64_t *)calloc((size_t)NB + 1, sizeof(int64_t));
    int64_t *ucnt = (int64_t *)calloc((size_t)NB + 1, sizeof(int64_t));
    if (!tmp || !hist || !boff || !ucnt) { free(keys); free(tmp); free(hist); free(boff); free(ucnt); return NULL; }
#pragma omp parallel num_threads(nth)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        const int64_t k0 = ntot * t / nth, k1 = ntot * (t + 1) / nth;
        int64_t *h = hist + (size_t)t * NB;
        for (int64_t k = k0; k < k1; ++k)
            if (keys[k] != SENT) h[keys[k] >> low]++;
#pragma omp barrier
#pragma omp single
        {
            int64_t acc = 0;
            for (int64_t b = 0; b < NB; ++b) {
                boff[b] = acc;
                for (int tt = 0; tt < nth; ++tt) {
                    int64_t c = hist[(size_t)tt * NB + b];
                    hist[(size_t)tt * NB + b] = acc;
                    acc += c;
                }
            }
            boff[NB] = acc;
        }
        for (int64_t k = k0; k < k1; ++k)
            if (keys[k] != SENT) tmp[h[keys[k] >> low]++] = keys[k];
    }
    int fail = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : fail)
    for (int64_t b = 0; b < NB; ++b) {
        const int64_t o = boff[b], c = boff[b + 1] - o;
        if (c > 1 && low > 0 && radix_sort_u64_buf(tmp + o, keys + o, c, low) != 0) fail = 1;
        int64_t nu = 0;
        for (int64_t k = 0; k < c; ++k)
            if (nu == 0 || tmp[o + k] != tmp[o + nu - 1]) tmp[o + nu++] = tmp[o + k];
        ucnt[b] = nu;
    }
    if (fail) { free(keys); free(tmp); free(hist); free(boff); free(ucnt); return NULL; }
    int64_t nu = 0;
    for (int64_t b = 0; b < NB; ++b) { int64_t c = ucnt[b]; ucnt[b] = nu; nu += c; }
    ucnt[NB] = nu;
    free(keys);
    sg_csr_t *m = (sg_csr_t *)calloc(1, sizeof(sg_csr_t));
    if (m) {
        m->n = n;
        m->nnz = nu;
        m->rowptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
        m->col = (int32_t *)malloc((size_t)(nu > 0 ? nu : 1) * sizeof(int32_t));
        m->val = (double *)malloc((size_t)(nu > 0 ? nu : 1) * sizeof(double));
        if (!m->rowptr || !m->col || !m->val) { sg_free(m); m = NULL; }
    }
    if (!m) { free(tmp); free(hist); free(boff); free(ucnt); return NULL; }
    const uint64_t cmask = ((uint64_t)1 << scale) - 1;
    /* per-row counts (rows of different buckets are disjoint), then the prefix sum */
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < NB; ++b) {
        const int64_t o = boff[b], c = ucnt[b + 1] - ucnt[b], d = ucnt[b];
        for (int64_t k = 0; k < c; ++k) {
            const uint64_t key = tmp[o + k];
            m->rowptr[(int64_t)(key >> scale) + 1]++;
            m->col[d + k] = (int32_t)(key & cmask);
        }
    }
    for (int64_t r = 0; r < n; ++r) m->rowptr[r + 1] += m->rowptr[r];
    free(tmp); free(hist); free(boff); free(ucnt);
    const uint64_t W = 0x57454947ull; /* "WEIG" */
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t k = m->rowptr[r]; k < m->rowptr[r + 1]; ++k) {
            uint64_t u = (uint64_t)r, v = (uint64_t)m->col[k];
            uint64_t lo = u < v ? u : v, hi = u < v ? v : u;
            uint64_t kk = 64 + (sg_h3(seed ^ W, lo, hi) >> 57);
            m->val[k] = (double)kk / 128.0;
        }
    }
    return m;
}

/* ------------------------------------------------------------------ */
/* Erdos-Renyi-like random symmetric COO with duplicates (exercises the
 * canonicaliser's duplicate summation). Sample e: u = floor(U0 n),
 * v = floor(U1 n), x = 2 U2 - 1 with Ud = U(h3(seed, e, d)); emits (u,v,x) and,
 * if u != v, (v,u,x) right after it. Returns the number of entries written
 * (<= 2*samples). */
int64_t sg_er_coo(int64_t n, int64_t samples, uint64_t seed, int64_t *ri, int32_t *ci,
                  double *v) {
    int64_t k = 0;
    for (int64_t e = 0; e < samples; ++e) {
        int64_t u = (int64_t)(sg_unit(sg_h3(seed, (uint64_t)e, 0)) * (double)n);
        int64_t w = (int64_t)(sg_unit(sg_h3(seed, (uint64_t)e, 1)) * (double)n);
        double x = 2.0 * sg_unit(sg_h3(seed, (uint64_t)e, 2)) - 1.0;
        if (u >= n) u = n - 1;
        if (w >= n) w = n - 1;
        ri[k] = u; ci[k] = (int32_t)w; v[k] = x; ++k;
        if (u != w) { ri[k] = w; ci[k] = (int32_t)u; v[k] = x; ++k; }
    }
    return k;
}

/* ------------------------------------------------------------------ */
/* Closed-form test matrices (BASELINE.json config 2).
 *   kind 0: Dirichlet tridiag(-1, 2, -1)          eig 2-2cos(pi k/(n+1)), k=1..n
 *   kind 1: path-graph Laplacian                  eig 2-2cos(pi k/n),     k=0..n-1
 *   kind 2: cycle Laplacian (n >= 3)              eig 2-2cos(2 pi k/n),   k=0..n-1 */
sg_csr_t *sg_tridiag(int kind, int64_t n) {
    if (n < 1 || (kind == 2 && n < 3)) return NULL;
    sg_csr_t *m = (sg_csr_t *)calloc(1, sizeof(sg_csr_t));
    if (!m) return NULL;
    int64_t cap = 3 * n;
    m->n = n;
    m->rowptr = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    m->col = (int32_t *)malloc((size_t)cap * sizeof(int32_t));
    m->val = (double *)malloc((size_t)cap * sizeof(double));
    if (!m->rowptr || !m->col || !m->val) { sg_free(m); return NULL; }
    int64_t k = 0;
    for (int64_t r = 0; r < n; ++r) {
        m->rowptr[r] = k;
        int64_t nb[3];
        double nv[3];
        int cnt = 0;
        double diag = 2.0;
        if (kind == 1) diag = (double)((r > 0) + (r < n - 1));
        if (kind == 2) {
            int64_t lft = (r + n - 1) % n, rgt = (r + 1) % n;
            /* sorted column order */
            int64_t cs[3] = {lft, r, rgt};
            double vs[3] = {-1.0, 2.0, -1.0};
            for (int i = 0; i < 3; ++i)
                for (int j = i + 1; j < 3; ++j)
                    if (cs[j] < cs[i]) {
                        int64_t t = cs[i]; cs[i] = cs[j]; cs[j] = t;
                        double tv = vs[i]; vs[i] = vs[j]; vs[j] = tv;
                    }
            for (int i = 0; i < 3; ++i) { nb[cnt] = cs[i]; nv[cnt] = vs[i]; ++cnt; }
        } else {
            if (r > 0) { nb[cnt] = r - 1; nv[cnt] = -1.0; ++cnt; }
            nb[cnt] = r; nv[cnt] = diag; ++cnt;
            if (r < n - 1) { nb[cnt] = r + 1; nv[cnt] = -1.0; ++cnt; }
        }
        for (int i = 0; i < cnt; ++i) {
            if (kind == 1 && n == 1) { nv[i] = 0.0; }
            m->col[k] = (int32_t)nb[i];
            m->val[k] = nv[i];
            ++k;
        }
    }
    m->rowptr[n] = k;
    m->nnz = k;
    return m;
}

/* 2-D grid (mesh / road-network class of Table I: hugetrace-00020, venturiLevel3,
 * *_osm, road_central). Vertex r = y * nx + x, 4-neighbour edges.
 *   kind 0: Dirichlet 5-point Laplacian (diagonal 4, off-diagonal -1, no drops);
 *           eigenvalues 4 - 2 cos(pi i/(nx+1)) - 2 cos(pi j/(ny+1)), i<=nx, j<=ny.
 *   kind 1: weighted graph Laplacian D - W: each grid edge {u, v} is kept unless
 *           U(h(seed, min, max)) < drop; weight k/128, k in [64, 191] from a second
 *           hash of the same pair (so both triangles hold identical bits); diagonal =
 *           sum of the kept weights (exact in f64/f32); isolated vertices have empty rows.
 * Columns are ascending within a row (r - nx, r - 1, r, r + 1, r + nx). */
static inline int grid_edge(uint64_t seed, double drop, int64_t u, int64_t v, double *w) {
    const int64_t a = u < v ? u : v, b = u < v ? v : u;
    if (sg_unit(sg_h3(seed, (uint64_t)a, (uint64_t)b)) < drop) return 0;
    *w = (double)(64 + (int)(sg_h3(seed ^ 0x5bd1e995ull, (uint64_t)a, (uint64_t)b) % 128)) / 128.0;
    return 1;
}

static int grid_row(int kind, int64_t nx, int64_t ny, double drop, uint64_t seed, int64_t r,
                    int32_t *col, double *val) {
    const int64_t x = r % nx, y = r / nx;
    int64_t nb[4];
    int c = 0;
    if (y > 0) nb[c++] = r - nx;
    if (x > 0) nb[c++] = r - 1;
    const int lower = c;
    if (x < nx - 1) nb[c++] = r + 1;
    if (y < ny - 1) nb[c++] = r + nx;
    int k = 0;
    double diag = 0.0;
    double wv[4];
    int keep[4];
    for (int i = 0; i < c; ++i) {
        if (kind == 0) { keep[i] = 1; wv[i] = 1.0; }
        else keep[i] = grid_edge(seed, drop, r, nb[i], &wv[i]);
        if (keep[i]) diag += wv[i];
    }
    if (kind == 0) diag = 4.0;
    for (int i = 0; i < lower; ++i)
        if (keep[i]) { if (col) { col[k] = (int32_t)nb[i]; val[k] = -wv[i]; } ++k; }
    if (kind == 0 || diag != 0.0) { if (col) { col[k] = (int32_t)r; val[k] = diag; } ++k; }
    for (int i = lower; i < c; ++i)
        if (keep[i]) { if (col) { col[k] = (int32_t)nb[i]; val[k] = -wv[i]; } ++k; }
    return k;
}

sg_csr_t *sg_grid2d(int kind, int64_t nx, int64_t ny, double drop, uint64_t seed) {
    if (nx < 1 || ny < 1 || nx * ny > 2147483647ll || (kind != 0 && kind != 1)) return NULL;
    const int64_t n = nx * ny;
    sg_csr_t *m = (sg_csr_t *)calloc(1, sizeof(sg_csr_t));
    if (!m) return NULL;
    m->n = n;
    m->rowptr = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    if (!m->rowptr) { sg_free(m); return NULL; }
    m->rowptr[0] = 0;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) m->rowptr[r + 1] = grid_row(kind, nx, ny, drop, seed, r, NULL, NULL);
    for (int64_t r = 0; r < n; ++r) m->rowptr[r + 1] += m->rowptr[r];
    m->nnz = m->rowptr[n];
    m->col = (int32_t *)malloc((size_t)(m->nnz > 0 ? m->nnz : 1) * sizeof(int32_t));
    m->val = (double *)malloc((size_t)(m->nnz > 0 ? m->nnz : 1) * sizeof(double));
    if (!m->col || !m->val) { sg_free(m); return NULL; }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r)
        grid_row(kind, nx, ny, drop, seed, r, m->col + m->rowptr[r], m->val + m->rowptr[r]);
    return m;
}
