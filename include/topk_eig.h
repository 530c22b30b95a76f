/*
 * topk_eig.h — C ABI of the B200-native Top-K sparse eigensolver hot path
 * (arXiv 2201.07498, "A Mixed Precision, Multi-GPU Design for Large-scale Top-K
 * Sparse Eigenproblems").
 *
 * The library computes the K largest-magnitude eigenvalues ("the largest in
 * modulo") and eigenvectors of a real symmetric sparse matrix M
 * with the paper's two-phase method (Fig. 1):
 *   phase 1  Lanczos, Algorithm 1: m iterations of
 *            SpMV (l.9) + alpha (l.10) + three-term recurrence (l.11) +
 *            full reorthogonalisation (l.12-18) + beta / normalise (l.6-7),
 *            rows partitioned by nnz;
 *   phase 2  Jacobi on the m x m tridiagonal T and the Ritz
 *            projection 𝒱V.
 * All steps run in hand-written sm_100a CUDA kernels owned by the handle.
 * Arithmetic is fp64 inside every kernel with vectors stored in the storage
 * dtype ("mixed precision": FDF = f32 storage, f64 compute).
 * Options beyond the paper's fixed-m iteration (all off by default; DESIGN.md
 * readings Q25-Q29): convergence-driven stop, thick restart, halo exchange,
 * periodic and partial reorthogonalisation (see topk_eig_opts_t).
 *
 * Conventions for every entry point
 *   - Returns topk_status_t; no exception or signal crosses the ABI. On error a
 *     message is available from topk_eig_last_error() (thread-local, valid until
 *     the next call on the same thread).
 *   - A CUDA or NCCL failure inside a handle makes it sticky: later calls on it
 *     return TOPK_E_STATE. Destroy it.
 *   - Pointers documented "host" must be host memory; "device" must be device
 *     memory of the handle's device. Inputs are borrowed (read during the call
 *     only); outputs are caller-owned buffers the library writes.
 *   - One handle may be used by one thread at a time (thread-compatible).
 *   - Breakdown (an exactly invariant Krylov subspace, beta ~ 0, reading Q7 of
 *     DESIGN.md) is NOT an error: TOPK_OK with info.breakdown = 1 and
 *     info.k_found < K; unused eigenvalue slots are NaN.
 */
#ifndef TOPK_EIG_H
#define TOPK_EIG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct topk_eig_s *topk_eig_t; /* opaque; owns device memory, streams, graph, NCCL comm */

typedef enum { TOPK_F64 = 0, TOPK_F32 = 1, TOPK_BF16 = 2 } topk_dtype_t;
typedef enum { TOPK_CSR = 0, TOPK_COO = 1 } topk_format_t;

typedef enum {
    TOPK_OK = 0,
    TOPK_E_INVALID = 1,       /* bad argument: K, m, n, dtype pair, null pointer, size          */
    TOPK_E_STRUCTURE = 2,     /* row_ptr not monotone / wrong ends, index out of range          */
    TOPK_E_NOT_SYMMETRIC = 3, /* symmetry check failed (structure or value bits)                */
    TOPK_E_NOMEM = 4,         /* host or device allocation failed                               */
    TOPK_E_CUDA = 5,          /* CUDA runtime error (handle becomes sticky)                     */
    TOPK_E_NCCL = 6,          /* NCCL error (handle becomes sticky)                             */
    TOPK_E_STATE = 7,         /* handle is sticky-failed or used out of order                   */
    TOPK_E_NODEVICE = 8       /* no CUDA device / wrong architecture (the library never falls back to the CPU) */
} topk_status_t;

/* The input matrix M ("Input Matrix M"; stored as COO in the paper,
 * PAPER.md:161). Borrowed during topk_eig_create only. Duplicated (row, col)
 * entries are summed in input order; columns are sorted within rows. */
typedef struct {
    topk_format_t format;
    int64_t n;              /* rows = cols; 1 <= n < 2^31                                        */
    int64_t nnz;            /* entries supplied (before duplicate summation)                     */
    const int64_t *row_ptr; /* CSR: host, n+1 entries, row_ptr[0]=0, non-decreasing, [n]=nnz      */
    const int64_t *row_idx; /* COO: host, nnz row indices in [0,n)                               */
    const int32_t *col_idx; /* host, nnz column indices in [0,n)                                 */
    const void *values;     /* host, nnz values of values_dtype; NULL = pattern (all ones)       */
    topk_dtype_t values_dtype; /* TOPK_F64 or TOPK_F32 (input representation)                 */
} topk_matrix_t;

/* Options. Zero-initialise, set struct_size = sizeof(topk_eig_opts_t), then set
 * the fields you need; 0 selects the documented default. */
typedef struct {
    uint32_t struct_size;
    int32_t krylov_dim;      /* m >= K Lanczos iterations; 0 -> K (the paper's "for i in 1, K", Alg.1 l.3) */
    int32_t reorth;          /* 1 full classical Gram-Schmidt (default; Alg.1 l.12-18 as full reorth,
                                reading Q3), 2 CGS twice, 3 partial (Simon's estimate decides per
                                iteration, reading Q29), -1 none (paper's optional mode) */
    int32_t num_parts;       /* G row partitions. Single process: G virtual ranks on
                                one device ("loopback"). Multi-process: must equal world. 0 -> 1     */
    int32_t device;          /* CUDA device ordinal of this process/handle                         */
    int32_t check_symmetry;  /* 0 default -> check; -1 skip (caller guarantees M = M^T). The check
                                compares the multiset of upper-triangle entries (position, value
                                bits) with the transposed lower ones through two 64-bit hash sums:
                                M = M^T always passes; an asymmetric M is rejected unless both sums
                                collide (~2^-128 for random-function hashes), i.e. the check is
                                probabilistic. One process per GPU: each rank hashes its own rows
                                and the sums are all-reduced (every rank returns the same status) */
    int32_t values_storage;  /* device dtype of matrix values; -1/0 default -> same as storage      */
    int32_t use_graph;       /* 0 default -> capture the solve as one CUDA graph; -1 -> eager launches */
    double breakdown_tol;    /* tau of reading Q7; 0 -> 1e-12 (f64), 1e-6 (f32), 1e-3 (bf16) storage */
    /* multi-process (one process per GPU, NCCL over NVLink) */
    int32_t rank;            /* this process's partition index g                                   */
    int32_t world;           /* number of processes; 0/1 -> single process                         */
    const void *nccl_id;     /* host, 128-byte ncclUniqueId from topk_eig_nccl_id() on rank 0     */
    int32_t profile;         /* 1 -> bracket every kernel of part 0 with CUDA events (recorded inside
                                the graph) so topk_eig_kernel_times() can report per-class device time */
    /* convergence-driven Krylov dimension (reading Q25; not in the
     * paper, which runs a fixed count, Alg.1 l.3): with conv_tol > 0, after iterations
     * i = c, 2c, ... (K <= i < krylov_dim) a Jacobi solve of T_i runs on the device and the
     * iteration stops at the first i where all K selected Ritz pairs have residual estimate
     * |beta_{i+1} s_{i,k}| <= conv_tol |theta_1|; krylov_dim becomes the cap. No host round trip:
     * the remaining launches of the graph see the stop flag and return at once. */
    double conv_tol;         /* 0 -> off (fixed krylov_dim iterations)                             */
    int32_t conv_check;      /* check period c; 0 -> K                                             */
    /* thick-restart Lanczos (Wu & Simon 2000, reading Q26; not in the
     * paper): with restart_keep = k > 0 the basis holds krylov_dim = m vectors; after each cycle the
     * k Ritz pairs of largest |theta| are kept (T becomes [[diag(theta), b], [b^T, tridiag]]) and the
     * iteration continues with steps k+1 .. m, up to max_restarts restarts; with conv_tol > 0 it stops
     * at the end of the first cycle whose K selected pairs meet the residual test. Requires
     * reorthogonalisation; K <= k <= min(m - 2, 256). Periodic conv_check tests are not used. */
    int32_t restart_keep;    /* 0 -> off                                                            */
    int32_t max_restarts;    /* restarts at most (the graph holds max_restarts + 1 cycles)           */
    /* vector exchange between parts (G > 1, reading Q27):
     * 0 -> every part receives the whole vector (ncclAllGather into a G * n_pad replica, the
     * paper's replicated v); 1 -> halo exchange: each part's SpMV reads a compact
     * vector [own slot | the remote entries its rows touch] and only those entries move (parts on
     * one device pull them; one process per GPU uses grouped ncclSend/ncclRecv; the multi-process
     * variant is built and covered by the host-logic tests but was not run on multi-GPU hardware) */
    int32_t exchange;
    /* periodic reorthogonalisation (reading Q28): with reorth = 1 and
     * reorth_period = p > 1 the full reorthogonalisation runs at the two consecutive iterations
     * kp and kp + 1 only (Grcar's periodic scheme); the others are the plain three-term step.
     * 0/1 -> every iteration. Not with thick restart. */
    int32_t reorth_period;
    /* kernel-path selection (no environment variables are read by the library; these
     * exist for A/B measurements and the tests that cover every path):
     * jacobi_path 0 -> auto (one CTA in shared memory for m <= 40, else a thread-block
     * cluster, else one CTA in global memory), 1 -> one CTA only, 2 -> cluster at any m;
     * jacobi_cluster 0 -> auto (8 CTAs, 16 from m = 96), 8 or 16 -> that size first;
     * restart_loop 0 -> thick-restart cycles in a CUDA-graph WHILE node when the solve is
     * captured, 1 -> unrolled cycles; ritz_path below. */
    int32_t jacobi_path;
    int32_t jacobi_cluster;
    int32_t restart_loop;
    /* Ritz output pass (a14) with compute dtype f64: 0 -> fp64 tensor cores (mma.sync
     * m8n8k4 f64) when the coefficients fit shared memory, 1 -> fp64 FMA on CUDA cores */
    int32_t ritz_path;
    /* overlapped vector exchange: with G > 1 and
     * exchange = 0 the SpMV runs as two passes, the own-slot columns first (they need nothing
     * from the peers), then the other columns and the epilogue; one process per GPU runs the
     * allgather of v_i on a second stream during the first pass. 0 -> on with one process per
     * GPU when a rank receives >= 64 MB per exchange ((G-1) n_pad storage bytes: the second
     * pass costs ~30-45 us per SpMV), off in one process; 1 -> on (also in one process: same
     * kernels and sums as the multi-process run); -1 -> off (one pass after the exchange). */
    int32_t overlap;
} topk_eig_opts_t;

typedef struct {
    int32_t k_found;          /* eigenpairs returned (= min(K, m') )                                */
    int32_t iterations;       /* m' Lanczos iterations completed                                    */
    int32_t breakdown;        /* 1 if Lanczos stopped early on beta <= tau * max(|alpha|, beta)      */
    int32_t jacobi_sweeps;
    int32_t jacobi_converged;
    int32_t num_parts;
    double beta_next;         /* beta_{m'+1} (reading Q6)                                           */
    double ms_solve;          /* device time of the whole solve (CUDA events)                       */
    int64_t bytes_model;      /* algorithmic HBM bytes of the solve on this part        */
    int64_t gpu_launches;     /* kernels launched by the solve (this part)                          */
    int32_t converged_stop;   /* 1 if conv_tol stopped the iteration early                         */
    int32_t conv_checks;      /* convergence checks enqueued per solve                             */
    int32_t restarts;         /* thick restarts done (iterations then counts every Lanczos step)   */
    int32_t reorth_passes;    /* reorth = 3: iterations that took the reorthogonalisation pass    */
    double ms_lanczos;        /* device time of v1 + the Lanczos iterations (phase 1)  */
    double ms_jacobi;         /* device time of the final Jacobi solve + top-K selection (a12-a13)  */
    double ms_ritz;           /* device time of the Ritz projection + output reordering (a14)      */
    int64_t bytes_nvlink;     /* one process per GPU: modelled bytes this rank receives over the
                                 interconnect per solve at the fixed m (the vector exchange, v1 +
                                 one per step, and the scalar allgathers); 0 in one process      */
} topk_eig_info_t;

/* Create a solver for M, K eigenpairs, storage/compute precision pair.
 *   storage : vector (and default value) storage dtype on the device
 *   compute : arithmetic dtype inside the kernels; compute >= storage precision.
 *             Supported (storage, compute): (F64,F64) "DDD", (F32,F64) "FDF",
 *             (F32,F32) "FFF", (BF16,F64); values_storage BF16 with F32 vectors.
 * Steps (DESIGN.md 8(a) rows a1-a4): canonicalise, check symmetry, partition by
 * nnz (rule P, reading Q15), build the per-part layout, upload to HBM.
 * Errors: TOPK_E_INVALID (K < 1, K > n, m < K, m > n, n >= 2^31, G * n_pad >= 2^31,
 * bad dtype pair, NULL pointers), TOPK_E_STRUCTURE, TOPK_E_NOT_SYMMETRIC,
 * TOPK_E_NOMEM, TOPK_E_CUDA, TOPK_E_NCCL, TOPK_E_NODEVICE. *out is NULL on error. */
topk_status_t topk_eig_create(topk_eig_t *out, const topk_matrix_t *A, int32_t K,
                              topk_dtype_t storage, topk_dtype_t compute,
                              const topk_eig_opts_t *opts);

/* Solve (DESIGN.md 8(a) rows a5-a15), host buffers.
 *   seed        : start vector u_r = 2 U(h3(seed, 0x7631, r)) - 1 (reading Q8), used if v1 == NULL
 *   v1          : host, NULL or n doubles: explicit start vector (normalised by the library)
 *   eigenvalues : host, K doubles out, ordered by (-|lambda|, -lambda); NaN past k_found
 *   eigenvectors: host, NULL or K*n out (vector k at [k*n, (k+1)*n)), dtype vec_dtype
 *                 (TOPK_F64 or TOPK_F32); unit norm, sign <y_k, v_1> > 0 (reading Q12).
 *                 Multi-process: each rank writes only its rows [b_g, b_{g+1}).
 *   residual_est: host, NULL or K doubles out: |beta_{m'+1} s_{m',k}|
 *   info        : host, NULL ok.
 * Synchronises the handle's stream. */
topk_status_t topk_eig_solve(topk_eig_t h, uint64_t seed, const double *v1, double *eigenvalues,
                             void *eigenvectors, topk_dtype_t vec_dtype, double *residual_est,
                             topk_eig_info_t *info);

/* Asynchronous solve on the handle's stream with device-resident outputs (no
 * host synchronisation): eigenvalues_dev (K doubles, device) and
 * eigenvectors_dev (NULL or K * n_local values of vec_dtype, device, vector k at
 * k * n_local) where n_local is this part's row count. Used for HBM-resident
 * timing. Call topk_eig_sync() before reading results or info. */
topk_status_t topk_eig_solve_async(topk_eig_t h, uint64_t seed, double *eigenvalues_dev,
                                   void *eigenvectors_dev, topk_dtype_t vec_dtype);
topk_status_t topk_eig_sync(topk_eig_t h, topk_eig_info_t *info);

/* The handle's CUDA stream (cudaStream_t as void*), for event timing by callers. */
void *topk_eig_stream(topk_eig_t h);

void topk_eig_destroy(topk_eig_t h); /* NULL-safe; frees device memory, graph, comm */
const char *topk_eig_last_error(void);

/* 128-byte NCCL unique id for a multi-process create (call on rank 0, broadcast). */
topk_status_t topk_eig_nccl_id(void *out128);

/* ---- host-only planning (no device needed): rule-P partition and per-part layout
 * (PAPER.md:125-128). Used by tests (CPU, gloo world_size 2) and by create. */
/* boundaries: host, G+1 int64 out. */
topk_status_t topk_eig_plan_partition(const int64_t *row_ptr, int64_t n, int32_t G,
                                      int64_t *boundaries);

/* Host-only per-part layout (rows a1, a3, a4 without a device): canonicalise A,
 * partition it by rule P into G parts and lay out part g exactly as
 * topk_eig_create uploads it, matrix values rounded to `values_storage`
 * (`storage` is validated only).
 *   sizes  (host, 9 int64 out): n_pad, n_rows, nnz, n_nonempty, nbig, nchunks,
 *          nslices, nitems, nphys
 *   logical CSR in degree order: rowptr (n_rows+1 int64), col (nnz int32 device
 *          column entries q*n_pad+pos), val (nnz doubles = stored values), perm
 *          (n_rows int32: original part-local row at each position)
 *   physical SpMV format: pcol (nphys int32), pval (nphys doubles), chunks (4
 *          int64 each: row, first physical nonzero, count, long id), sell (2
 *          int64 per slice: base, width), items (2 int32 per SELL work item:
 *          first, end slice). Offsets are 64-bit: a part may hold >= 2^31
 *          nonzeros.
 * Every array pointer may be NULL. Used by the multi-process CPU tests (each
 * rank plans its own part). Errors as in create. */
topk_status_t topk_eig_plan_layout(const topk_matrix_t *A, int32_t G, int32_t g, topk_dtype_t storage,
                                   topk_dtype_t values_storage, int64_t *sizes, int64_t *rowptr,
                                   int32_t *col, double *val, int32_t *perm, int32_t *pcol, double *pval,
                                   int64_t *chunks, int64_t *sell, int32_t *items);

/* Memory runtime (mem_pool.h): device blocks freed by topk_eig_destroy are cached
 * per device and reused by later handles (no cudaMalloc/cudaFree on the create/
 * destroy path after the first handle); large host blocks of the create-time layout
 * arrays are cached the same way (no page faults on fresh memory per create).
 * Returns every cached, unused device and host block to the driver / the C heap;
 * returns the bytes released. Thread-safe; live handles are unaffected. */
size_t topk_eig_trim_pool(void);

/* Host-only: the symmetry check's four wrapping 64-bit hash sums over rows [r0, r1) of
 * the canonical matrix (row a2, reading Q17): sums[0], sums[1] over the entries (r, c, v)
 * with c > r, sums[2], sums[3] over the transposed entries with c < r (key (min, max),
 * value bits). The sums are additive over row ranges: one process per GPU hashes its
 * own rows and the ranks add their sums (create does this with an NCCL all-reduce);
 * M = M^T passes always, an asymmetric M only on a double 64-bit collision. sums: host,
 * 4 uint64 out. Errors as in create. */
topk_status_t topk_eig_plan_symmetry(const topk_matrix_t *A, int64_t r0, int64_t r1, uint64_t *sums);

/* Host-only halo plan of part g of G (reading Q27): the
 * remote entries part g's SpMV reads, grouped by owner q in ascending owner position,
 * exactly as topk_eig_create with opts.exchange = 1 lays them out after the own slot.
 *   n_halo (host, 1 int64 out), off (host, NULL or G+1 int64: owner q's entries are
 *   [off[q], off[q+1])), pos (host, NULL or n_halo int32: position in the owner's slot).
 * Used by the multi-process CPU tests to check the request/send lists. Errors as in create. */
topk_status_t topk_eig_plan_halo(const topk_matrix_t *A, int32_t G, int32_t g, int64_t *n_halo, int64_t *off,
                                 int32_t *pos);

/* Per kernel class device time of the last solve (requires opts.profile = 1):
 * class 0 v1, 1 spmv, 2 step, 3 correct, 4 jacobi, 5 ritz pass 0 (norms), 6 ritz pass 1 (output),
 * 7 unpermute (output back to the original row order).
 * ms (host, 8 doubles): summed milliseconds; launches (host, 8 int32): launch counts.
 * Events bracket each launch on the handle's stream (the stream the kernels run on). */
topk_status_t topk_eig_kernel_times(topk_eig_t h, double *ms, int32_t *launches);

/* ---- test/debug exports (same ABI; documented unstable) ---- */
/* boundaries: host, G+1 int64 out */
topk_status_t topk_eig_export_partition(topk_eig_t h, int64_t *boundaries);
/* Part p (0 <= p < local parts) logical layout, reassembled from the uploaded physical
 * arrays: rowptr host (n_p+1 int64, degree row order), col host (z_p int32 device column
 * entries, see topk_eig_plan_layout), val host (z_p doubles = stored values), n_pad out,
 * sizes out (n_p, z_p). Any pointer may be NULL to query sizes only. */
topk_status_t topk_eig_export_layout(topk_eig_t h, int32_t part, int64_t *rowptr, int32_t *col,
                                     double *val, int64_t *n_pad, int64_t *n_rows,
                                     int64_t *nnz);
/* After a solve: alpha (m' doubles), beta (m'+1 doubles, beta[0] = 0), theta_all
 * (m' doubles, Jacobi order), m_found out. Any pointer may be NULL. */
topk_status_t topk_eig_export_tridiag(topk_eig_t h, double *alpha, double *beta,
                                      double *theta_all, int32_t *m_found);
/* After a solve: the stored Lanczos basis of part p as doubles: V[j * n_p + r] =
 * s_j * u_j[r] for j < m'+1 (m'+1 columns when no breakdown), i.e. the
 * normalised v_{j+1} (host, (m'+1) * n_p doubles). */
topk_status_t topk_eig_export_basis(topk_eig_t h, int32_t part, double *V, int32_t *ncols);
/* After a solve: the stored basis columns of part p WITHOUT the deferred scale s_j,
 * converted exactly from the storage dtype to double: U[j * n_p + r] = u_j[r]. Column 0
 * is the unnormalised start vector u_r = 2 U(h3(seed, 0x7631, row0 + r)) - 1 (reading
 * Q8) rounded once to the storage dtype, the quantity the parity
 * contract compares bit for bit with the oracle's orc_v1. Same sizes and
 * NULL rules as topk_eig_export_basis. */
topk_status_t topk_eig_export_basis_raw(topk_eig_t h, int32_t part, double *U, int32_t *ncols);
/* One SpMV y = M x through the device kernel on part-local rows (x, y host, n
 * doubles, global indexing; x is rounded to the storage dtype first, y is the
 * fp64 row sums before storage rounding). */
topk_status_t topk_eig_debug_spmv(topk_eig_t h, const double *x, double *y);

#ifdef __cplusplus
}
#endif
#endif /* TOPK_EIG_H */
