/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the Top-K sparse
 * eigensolver hot path of arXiv 2201.07498 ("A Mixed Precision, Multi-GPU
 * Design for Large-scale Top-K Sparse Eigenproblems").
 *
 * *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library. The product path (paper_2201_07498_b200/) never touches it; the two
 * share no code, headers or helpers (the seeded matrix generators in synthgen/
 * are the only shared module, and they hold none of the method's arithmetic).
 *
 * Single thread, fp64 everywhere, sequential sums in index order, no blocking,
 * no fusion, no SIMD intrinsics. Every function cites the passage it follows:
 *   PAPER.md:N  = line N of /root/reference/PAPER.md (the paper's LaTeX source)
 *   Alg.1 l.N   = line N of the paper's Algorithm 1 (numbering: SURVEY.md 0)
 *   Qn          = reading n of the paper listed in DESIGN.md "Readings".
 *
 * Pins (tests/test_oracle_*.py): every function below is pinned against
 * something other than itself (dense eigh, closed forms, brute force, printed
 * examples, invariants). See DESIGN.md "Oracle pins". No function here is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_E_INVALID 1
#define ORC_E_STRUCTURE 2
#define ORC_E_NOMEM 4

/* ------------------------------------------------------------------------ */
/* O1. Canonicalisation COO -> CSR (SPEC.md:58-66 used for the interface;
 * the paper stores M as COO, and runs an SpMV on it, Alg.1 l.9;
 * reading Q18: CSR is the compute format).
 * Entries are grouped by row keeping input order (counting placement), then
 * each row is insertion-sorted by column (stable), then equal (row, col)
 * entries are summed in input order. Returns the canonical nnz, or -code. */
int64_t orc_coo_to_csr(int64_t n, int64_t nnz, const int64_t *ri, const int32_t *ci,
                       const double *v, int64_t *rowptr, int32_t *col, double *val) {
    if (n < 0 || nnz < 0) return -ORC_E_INVALID;
    for (int64_t k = 0; k < nnz; ++k)
        if (ri[k] < 0 || ri[k] >= n || ci[k] < 0 || (int64_t)ci[k] >= n) return -ORC_E_STRUCTURE;
    int64_t *cnt = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t *fill = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    if (!cnt || !fill) { free(cnt); free(fill); return -ORC_E_NOMEM; }
    for (int64_t k = 0; k < nnz; ++k) cnt[ri[k] + 1]++;
    for (int64_t r = 0; r < n; ++r) cnt[r + 1] += cnt[r];
    /* stable placement by row */
    for (int64_t k = 0; k < nnz; ++k) {
        int64_t pos = cnt[ri[k]] + fill[ri[k]]++;
        col[pos] = ci[k];
        val[pos] = v[k];
    }
    /* per row: stable insertion sort by column, then sum duplicates in order */
    int64_t out = 0;
    for (int64_t r = 0; r < n; ++r) {
        int64_t b = cnt[r], e = cnt[r + 1];
        for (int64_t i = b + 1; i < e; ++i) {
            int32_t c = col[i];
            double x = val[i];
            int64_t j = i - 1;
            while (j >= b && col[j] > c) { col[j + 1] = col[j]; val[j + 1] = val[j]; --j; }
            col[j + 1] = c;
            val[j + 1] = x;
        }
        rowptr[r] = out;
        for (int64_t i = b; i < e; ++i) {
            if (out > rowptr[r] && col[out - 1] == col[i]) {
                val[out - 1] = val[out - 1] + val[i];
            } else {
                col[out] = col[i];
                val[out] = val[i];
                ++out;
            }
        }
    }
    rowptr[n] = out;
    free(cnt);
    free(fill);
    return out;
}

/* O1 (symmetry). Lanczos needs M = M^T (PAPER.md:30 "real-valued", :35).
 * Canonical CSR in; every (r,c,x) must have a (c,r,x') with identical bits. */
int orc_is_symmetric(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val) {
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
            int64_t c = col[k];
            int64_t lo = rowptr[c], hi = rowptr[c + 1] - 1, found = -1;
            while (lo <= hi) {
                int64_t mid = lo + (hi - lo) / 2;
                if (col[mid] == r) { found = mid; break; }
                if (col[mid] < r) lo = mid + 1; else hi = mid - 1;
            }
            if (found < 0) return 0;
            if (memcmp(&val[found], &val[k], sizeof(double)) != 0) return 0;
        }
    }
    return 1;
}

/* ------------------------------------------------------------------------ */
/* O2. nnz-balanced row partition ("The input matrix is partitioned
 * by balancing the number of non-zero elements in each partition"; reading Q15):
 * contiguous row ranges, each >= 1 row, minimising the maximum part nnz; among
 * optimal splits the lexicographically smallest boundary vector.
 *   B* = min B such that a left-to-right greedy (start a new part when the next
 *        row would overflow B) needs <= G parts  (binary search on B);
 *   b[G] = n; for k = G-1..1: b[k] = max(first j with rowptr[j] >= rowptr[b[k+1]] - B*, k);
 *   b[0] = 0.                                                                   */
static int64_t greedy_parts(int64_t n, const int64_t *rowptr, int64_t B) {
    int64_t parts = 1, start = 0;
    for (int64_t r = 0; r < n; ++r) {
        if (rowptr[r + 1] - rowptr[r] > B) return INT64_MAX;
        if (rowptr[r + 1] - rowptr[start] > B) { ++parts; start = r; }
    }
    return parts;
}

int orc_partition(int64_t n, const int64_t *rowptr, int32_t G, int64_t *b) {
    if (G < 1 || n < G) return ORC_E_INVALID;
    int64_t lo = 0, hi = rowptr[n];
    for (int64_t r = 0; r < n; ++r)
        if (rowptr[r + 1] - rowptr[r] > lo) lo = rowptr[r + 1] - rowptr[r];
    while (lo < hi) { /* smallest feasible B in [max row nnz, nnz] */
        int64_t mid = lo + (hi - lo) / 2;
        if (greedy_parts(n, rowptr, mid) <= G) hi = mid; else lo = mid + 1;
    }
    int64_t Bs = lo;
    b[G] = n;
    for (int32_t k = G - 1; k >= 1; --k) {
        int64_t target = rowptr[b[k + 1]] - Bs;
        int64_t j = 0;
        while (rowptr[j] < target) ++j; /* first j with rowptr[j] >= target */
        b[k] = j > k ? j : k;
    }
    b[0] = 0;
    return ORC_OK;
}

/* Storage-dtype rounding (reading Q14/Q22): round-to-nearest-even once, straight
 * from f64. dtype 0 = f64 (identity), 1 = f32, 2 = bf16 (8 significant bits). */
static double round_to_dtype(double x, int dtype) {
    if (dtype == 0) return x;
    if (dtype == 1) return (double)(float)x;
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    double m = frexp(x, &e);           /* x = m 2^e, 0.5 <= |m| < 1 */
    double r = rint(ldexp(m, 8));      /* 8 significant bits, ties to even */
    return ldexp(r, e - 8);
}

/* O2 (layout). Per-partition CSR of partition g (rows of M_g;
 * v_i replicated): rows of the part in degree order (orc_positions), local
 * rowptr rebased to 0; columns remapped into the padded replica
 * c' = g(c) * n_pad + pos[c] with n_pad = round_up(max_g n_g, 64) (SURVEY.md
 * 8(e) "v1 = padded"); values rounded to the
 * storage dtype (out_val receives the rounded values as f64, their exact
 * value); out_perm[p] = part-local original row at position p. */
/* (degree-descending comparator shared by the layout functions below) */
static const int64_t *g_deg_rowptr;
static int cmp_deg_desc(const void *pa, const void *pb) {
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    int64_t da = g_deg_rowptr[a + 1] - g_deg_rowptr[a], db = g_deg_rowptr[b + 1] - g_deg_rowptr[b];
    if (da != db) return da > db ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}


/* Degree order (a layout choice, not a paper construct):
 * inside part q the rows are sorted by (degree descending, index ascending);
 * empty rows therefore come last. pos[r] = position of global row r inside its
 * part. */
int orc_positions(int64_t n, const int64_t *rowptr, int32_t G, const int64_t *b, int32_t *pos) {
    (void)n;
    for (int32_t q = 0; q < G; ++q) {
        int64_t nr = b[q + 1] - b[q];
        int64_t *rows = (int64_t *)malloc((size_t)(nr > 0 ? nr : 1) * sizeof(int64_t));
        if (!rows) return ORC_E_NOMEM;
        for (int64_t i = 0; i < nr; ++i) rows[i] = b[q] + i;
        g_deg_rowptr = rowptr;
        qsort(rows, (size_t)nr, sizeof(int64_t), cmp_deg_desc);
        for (int64_t i = 0; i < nr; ++i) pos[rows[i]] = (int32_t)i;
        free(rows);
    }
    return ORC_OK;
}

int64_t orc_layout(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val,
                   int32_t G, const int64_t *b, int32_t g, int dtype, const int32_t *pos,
                   int64_t *out_rowptr, int32_t *out_col, double *out_val, int32_t *out_perm) {
    (void)n;
    int64_t npad = 0;
    for (int32_t p = 0; p < G; ++p)
        if (b[p + 1] - b[p] > npad) npad = b[p + 1] - b[p];
    npad = (npad + 63) / 64 * 64;
    for (int64_t r = b[g]; r < b[g + 1]; ++r) out_perm[pos[r]] = (int32_t)(r - b[g]);
    int64_t o = 0;
    out_rowptr[0] = 0;
    for (int64_t p = 0; p < b[g + 1] - b[g]; ++p) {
        int64_t r = b[g] + out_perm[p];
        for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k, ++o) {
            int64_t c = col[k];
            int32_t owner = 0;
            while (!(c >= b[owner] && c < b[owner + 1])) ++owner;
            uint32_t cc = (uint32_t)(owner * npad + pos[c]);
            out_col[o] = (int32_t)cc;
            out_val[o] = round_to_dtype(val[k], dtype);
        }
        out_rowptr[p + 1] = o;
    }
    return npad;
}


/* ------------------------------------------------------------------------ */
/* O3. Random start vector ("L2-normalized random vector v_1";
 * :205 "random initialization"; reading Q8): u_r = 2 U(h3(seed, 0x7631, r)) - 1
 * with the splitmix64 finaliser mix64, h3(s,a,b) = mix64(mix64(mix64(s)^a)^b),
 * U(x) = (x >> 11) 2^-53. Unnormalised; the caller normalises. */
static uint64_t orc_mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void orc_v1(uint64_t seed, int64_t n, double *u) {
    for (int64_t r = 0; r < n; ++r) {
        uint64_t h = orc_mix64(orc_mix64(orc_mix64(seed) ^ 0x7631ull) ^ (uint64_t)r);
        u[r] = 2.0 * ((double)(h >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
    }
}

/* ------------------------------------------------------------------------ */
/* Alg.1 l.9: SpMV y = M x, row by row, k ascending within the row. */
void orc_spmv(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val,
              const double *x, double *y) {
    for (int64_t r = 0; r < n; ++r) {
        double s = 0.0;
        for (int64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) s += val[k] * x[col[k]];
        y[r] = s;
    }
}

static double dot(int64_t n, const double *a, const double *b) {
    double s = 0.0;
    for (int64_t r = 0; r < n; ++r) s += a[r] * b[r];
    return s;
}

/* ------------------------------------------------------------------------ */
/* One iteration i (1-based) of Algorithm 1, l.5-18, on explicit state:
 * Vw holds v_1..v_{i-1} (column-major, v_1 already normalised), vn holds v_nxt
 * of iteration i-1, vt is scratch for v_tmp. Writes v_i, alpha_i, beta_i and the
 * new v_nxt; *tscale is max(|alpha|, beta) so far (reading Q7). Returns 1 on
 * breakdown (beta_i <= tau * tscale), else 0. orc_lanczos is this in a loop;
 * bench.py's reference arm times single iterations of it. */
int orc_lanczos_iter(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val,
                     int32_t i, int32_t reorth, double tau, double *Vw, double *vt, double *vn,
                     double *alpha, double *beta, double *tscale) {
    double *vi = Vw + (size_t)(i - 1) * n;
    if (i != 1) {                               /* l.5 */
        double bi = sqrt(dot(n, vn, vn));       /* l.6 beta_i = ||v_nxt|| */
        beta[i - 1] = bi;
        if (bi <= tau * *tscale) return 1;
        for (int64_t r = 0; r < n; ++r) vi[r] = vn[r] / bi; /* l.7 */
        if (bi > *tscale) *tscale = bi;
    }
    orc_spmv(n, rowptr, col, val, vi, vt);          /* l.9 v_t = M v_i */
    double ai = dot(n, vi, vt);                     /* l.10 alpha_i */
    alpha[i - 1] = ai;
    if (fabs(ai) > *tscale) *tscale = fabs(ai);
    const double *vprev = (i > 1) ? Vw + (size_t)(i - 2) * n : NULL;
    double bi = beta[i - 1];
    for (int64_t r = 0; r < n; ++r)                 /* l.11 */
        vn[r] = vt[r] - ai * vi[r] - (vprev ? bi * vprev[r] : 0.0);
    if (reorth) {                                   /* l.12-18 (Q3) */
        for (int32_t j = 1; j <= i; ++j) {
            const double *vj = Vw + (size_t)(j - 1) * n;
            double o = dot(n, vj, vn);
            for (int64_t r = 0; r < n; ++r) vn[r] -= o * vj[r];
        }
    }
    return 0;
}

/* O4-O6. Lanczos, Algorithm 1, m iterations (reading Q5:
 * m >= K; m = K is the paper's "for i in 1, K", l.3).
 *   v1     : start vector (normalised here, "L2-normalized")
 *   reorth : 1 = full reorthogonalisation of v_nxt against v_1..v_i by modified
 *            Gram-Schmidt, one pass, alpha not corrected (l.12-18, readings Q3,Q4);
 *            0 = none.
 *   tau    : breakdown threshold (reading Q7): stop when beta_i <= tau * Tscale,
 *            Tscale = max(|alpha_1..alpha_{i-1}|, beta_2..beta_{i-1}).
 * Outputs (0-based): alpha[k] = alpha_{k+1} (k < m'); beta[0] = beta_1 = 0,
 * beta[k] = beta_{k+1} (k <= m'): beta[m'] is beta_{m'+1} (reading Q6, the
 * residual-estimate factor; at breakdown it is the tiny beta that stopped it).
 * V (n*m, optional) receives v_1..v_m' column by column (V[j*n + r]).
 * Returns m' (number of completed iterations); *breakdown = 1 if stopped early. */
int64_t orc_lanczos(int64_t n, const int64_t *rowptr, const int32_t *col, const double *val,
                    const double *v1, int32_t m, int32_t reorth, double tau, double *alpha,
                    double *beta, double *V, int32_t *breakdown) {
    double *Vw = V;
    int own = 0;
    if (!Vw) {
        Vw = (double *)malloc((size_t)n * (size_t)(m > 0 ? m : 1) * sizeof(double));
        own = 1;
    }
    double *vt = (double *)malloc((size_t)n * sizeof(double));   /* v_tmp (Q2) */
    double *vn = (double *)malloc((size_t)n * sizeof(double));   /* v_nxt (Q2) */
    if (!Vw || !vt || !vn) { if (own) free(Vw); free(vt); free(vn); return -ORC_E_NOMEM; }
    *breakdown = 0;
    /* v_1 = v1 / ||v1|| */
    double nrm = sqrt(dot(n, v1, v1));
    for (int64_t r = 0; r < n; ++r) Vw[r] = v1[r] / nrm;
    beta[0] = 0.0; /* l.2: beta_1 <- 0 */
    double tscale = 0.0;
    int64_t done = 0;
    for (int32_t i = 1; i <= m; ++i) {           /* l.3 */
        if (orc_lanczos_iter(n, rowptr, col, val, i, reorth, tau, Vw, vt, vn, alpha, beta, &tscale)) {
            *breakdown = 1;
            break;
        }
        done = i;
    }
    if (!*breakdown) beta[done] = sqrt(dot(n, vn, vn)); /* Q6: beta_{m+1} */
    if (own) free(Vw);
    free(vt);
    free(vn);
    return done;
}

/* ------------------------------------------------------------------------ */
/* O7. Jacobi eigenvalue algorithm on the small symmetric T (PAPER.md:114-115,
 * citing Rutishauser 1966; reading Q10). Cyclic-by-row ordering
 * (p = 0..m-2, q = p+1..m-1). A rotation J(p,q) with
 *   zeta = (a_qq - a_pp) / (2 a_pq), t = sgn(zeta) / (|zeta| + sqrt(1 + zeta^2))
 *   (sgn(0) = 1), c = 1/sqrt(1+t^2), s = t c
 * annihilates a_pq:  A <- J^T A J, S <- S J, then a_pq = a_qp = 0 exactly.
 * An off-diagonal entry is negligible (set to 0, no rotation) when
 *   |a_pq| <= eps sqrt(|a_pp a_qq|)  or  |a_pq| <= eps^2 ||A||_F,  eps = 2^-52.
 * Stops after a sweep with no rotation (converged) or max_sweeps sweeps.
 * A is m*m row-major (destroyed), theta[m] = final diagonal, S m*m row-major
 * with column k the eigenvector of theta[k]. Returns 1 if converged. */
int orc_jacobi(int32_t m, double *A, double *theta, double *S, int32_t max_sweeps,
               int32_t *sweeps) {
    const double eps = 2.220446049250313e-16;
    double fro = 0.0;
    for (int64_t k = 0; k < (int64_t)m * m; ++k) fro += A[k] * A[k];
    fro = sqrt(fro);
    for (int32_t p = 0; p < m; ++p)
        for (int32_t q = 0; q < m; ++q) S[p * m + q] = (p == q) ? 1.0 : 0.0;
    int converged = 0;
    int32_t sw = 0;
    while (sw < max_sweeps) {
        int rotated = 0;
        for (int32_t p = 0; p < m - 1; ++p) {
            for (int32_t q = p + 1; q < m; ++q) {
                double apq = A[p * m + q];
                double app = A[p * m + p], aqq = A[q * m + q];
                if (fabs(apq) <= eps * sqrt(fabs(app * aqq)) || fabs(apq) <= eps * eps * fro) {
                    A[p * m + q] = 0.0;
                    A[q * m + p] = 0.0;
                    continue;
                }
                rotated = 1;
                double zeta = (aqq - app) / (2.0 * apq);
                double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = t * c;
                /* A <- A J : columns p, q */
                for (int32_t k = 0; k < m; ++k) {
                    double akp = A[k * m + p], akq = A[k * m + q];
                    A[k * m + p] = c * akp - s * akq;
                    A[k * m + q] = s * akp + c * akq;
                }
                /* A <- J^T A : rows p, q */
                for (int32_t k = 0; k < m; ++k) {
                    double apk = A[p * m + k], aqk = A[q * m + k];
                    A[p * m + k] = c * apk - s * aqk;
                    A[q * m + k] = s * apk + c * aqk;
                }
                A[p * m + q] = 0.0;
                A[q * m + p] = 0.0;
                /* S <- S J */
                for (int32_t k = 0; k < m; ++k) {
                    double skp = S[k * m + p], skq = S[k * m + q];
                    S[k * m + p] = c * skp - s * skq;
                    S[k * m + q] = s * skp + c * skq;
                }
            }
        }
        ++sw;
        if (!rotated) { converged = 1; break; }
    }
    for (int32_t k = 0; k < m; ++k) theta[k] = A[k * m + k];
    *sweeps = sw;
    return converged;
}

/* ------------------------------------------------------------------------ */
/* O8. Top-K selection "largest (in modulo)" (reading Q9):
 * order by (-|theta|, -theta), equal keys by index; keep min(K, m). */
static int key_before(const double *th, int32_t a, int32_t b) {
    double fa = fabs(th[a]), fb = fabs(th[b]);
    if (fa != fb) return fa > fb;
    if (th[a] != th[b]) return th[a] > th[b];
    return a < b;
}

int32_t orc_select(int32_t m, const double *theta, int32_t K, int32_t *idx) {
    int32_t *ord = (int32_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int32_t));
    if (!ord) return -ORC_E_NOMEM;
    for (int32_t i = 0; i < m; ++i) ord[i] = i;
    for (int32_t i = 1; i < m; ++i) { /* insertion sort by the key */
        int32_t x = ord[i], j = i - 1;
        while (j >= 0 && key_before(theta, x, ord[j])) { ord[j + 1] = ord[j]; --j; }
        ord[j + 1] = x;
    }
    int32_t kk = K < m ? K : m;
    for (int32_t i = 0; i < kk; ++i) idx[i] = ord[i];
    free(ord);
    return kk;
}

/* O9. Ritz vectors y_k = V s_k ("The eigenvectors of M are given by
 * 𝒱V"), sign fixed so that the first nonzero entry of s_k is positive (reading
 * Q12: <y_k, v_1> > 0), then normalised. V is n*mm column-major
 * (V[j*n + r]); S is mm*mm row-major (column k = eigenvector); Y is K*n. */
void orc_ritz(int64_t n, int32_t mm, const double *V, const double *S, int32_t K,
              const int32_t *idx, double *Y) {
    for (int32_t k = 0; k < K; ++k) {
        int32_t c = idx[k];
        double sg = 1.0;
        for (int32_t j = 0; j < mm; ++j) {
            double s = S[j * mm + c];
            if (s != 0.0) { sg = s > 0.0 ? 1.0 : -1.0; break; }
        }
        double *y = Y + (size_t)k * n;
        for (int64_t r = 0; r < n; ++r) {
            double acc = 0.0;
            for (int32_t j = 0; j < mm; ++j) acc += S[j * mm + c] * V[(size_t)j * n + r];
            y[r] = sg * acc;
        }
        double nr = sqrt(dot(n, y, y));
        for (int64_t r = 0; r < n; ++r) y[r] /= nr;
    }
}
