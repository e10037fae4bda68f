/*
 * ebv.h — C ABI of libebv.so, the B200 (sm_100a) implementation of the hot
 * path of the "Equal bi-Vectorized" (EbV) method, arXiv 1907.05767.
 *
 * Citations: P:<line> = PAPER.md (the paper text), DESIGN.md = this repo's
 * design notes (readings R1..R17 of the garbled passages), SURVEY §8 = the
 * scope table (rows A1-A13 and the "next" rows f1-f4).
 *
 * The problem statement followed by every call (Eq 1):
 *     AX = B  <=>  (LU)X = B  <=>  L(UX) = B  <=>  LY = B, then UX = Y.
 * A is factored without pivoting into a unit lower triangular L and an upper
 * triangular U (Doolittle; Eq 3, reading R1) by the per-step
 * recurrences of Eq 6:
 *     l_ik = a_ik / a_kk            (Eq 6-a, the L_(k) column vector)
 *     u_kj = a_kj                   (Eq 6-b, the U_(k) row vector, reading R1)
 *     a_ij <- a_ij - l_ik u_kj      (Eq 6-c, the rank-1 update of A^(k))
 * for a diagonally dominant A ("diagonal dominant shape").  Every
 * entry is produced as the fma chain over ascending k followed (for L) by a
 * correctly rounded division — the canonical order of DESIGN.md, which makes
 * the results bitwise identical to the serial oracle.
 *
 * Conventions shared by all calls
 *   - Matrices are column-major: a(i, j) = A[i + j*lda], lda >= n.  The
 *     factorization is packed in place: strict lower triangle = L multipliers
 *     (unit diagonal implicit), diagonal + upper triangle = U.
 *   - All matrix / vector / info pointers are DEVICE pointers owned by the
 *     caller (except the host matrix of ebv_lu_factor_host); the library
 *     never frees them.  The library owns only its context (workspace,
 *     streams, events, NCCL communicator).
 *   - Calls are asynchronous on the caller's `stream` (a cudaStream_t passed
 *     as void*; NULL = legacy default stream).  The library never
 *     synchronizes the caller's stream.
 *   - A context's workspace (pivot floor, arrival counters, solve flags,
 *     batched scratch) is shared by its calls: calls on one context must be
 *     ordered (one stream, or streams ordered by events); use one context
 *     per concurrent stream / host thread.
 *   - Host-detectable argument errors return EBV_ERR_INVALID_VALUE before
 *     anything is launched.  CUDA launch / runtime failures return
 *     EBV_ERR_CUDA; ebv_last_error() gives a one-line description.
 *   - A singular / small pivot is never a return code: it is reported through
 *     the device-side info word(s) (LAPACK getrf convention): 0, or the first
 *     1-based step r with |u_rr| <= tau.  The factorization always runs to
 *     completion; outputs are unspecified (may hold Inf/NaN) when info != 0.
 *   - tau: pivot floor.  tau >= 0 is used as is (0 = exact-zero check only);
 *     tau < 0 selects the default n * DBL_EPSILON * ||A||_inf (reading R9),
 *     computed on the device by a norm pre-pass.
 */
#ifndef EBV_H_
#define EBV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  EBV_SUCCESS = 0,
  EBV_ERR_INVALID_VALUE = 1,  /* bad size / stride / NULL pointer            */
  EBV_ERR_SINGULAR_PIVOT = 2, /* never returned by the async calls; for
                                 callers that map a nonzero info word        */
  EBV_ERR_CUDA = 3,           /* a CUDA runtime error (see ebv_last_error)    */
  EBV_ERR_NCCL = 4,           /* reserved for the multi-GPU context           */
  EBV_ERR_NOT_SUPPORTED = 5,  /* valid but unsupported (e.g. batched n > 64)  */
  EBV_ERR_ALLOC = 6           /* workspace allocation failed                  */
} ebv_status_t;

/* Opaque context: device, workspace, auxiliary streams/events, options. */
typedef struct ebv_context* ebv_context_t;

/* Which factorization path ebv_lu_factor takes.
 *   EBV_PATH_VECTOR  — the paper's vector-level elimination (Eq 6 step by
 *                      step) as one persistent kernel: blocks of up
 *                      to 8 consecutive columns, EbV-paired blocks (J, Nb-1-J)
 *                      (Eq 7) dealt to CTAs and resident in shared
 *                      memory; the owner of block J factors it and releases
 *                      one flag, every CTA applies its L_(k) vectors to its
 *                      later columns.  n <= EBV_VECTOR_MAX_N.
 *   EBV_PATH_BLOCKED — right-looking blocked form of the same recurrences:
 *                      the trailing rank-nb updates run as FP64 tensor-core
 *                      (DMMA) contractions, triangular blocks by row/column-
 *                      parallel substitution, lookahead on a side stream.
 *   EBV_PATH_LEFT    — left-looking blocked form (block J takes all earlier
 *                      panels' updates — a trsm with L[0:c, 0:c] and one DMMA
 *                      contraction — before its own panel); it can stream a
 *                      host-resident matrix (ebv_lu_factor_host) but its
 *                      per-block triangular solves are launch-heavy: slower
 *                      than EBV_PATH_BLOCKED at every n measured.
 *   EBV_PATH_AUTO    — the blocked (right-looking) path.
 * All paths give bitwise the same factors.                                   */
typedef enum { EBV_PATH_AUTO = 0, EBV_PATH_VECTOR = 1, EBV_PATH_BLOCKED = 2, EBV_PATH_LEFT = 3 } ebv_path_t;

#define EBV_VECTOR_MAX_N 1536
#define EBV_BATCHED_MAX_N 64          /* register-resident kernels (one or two systems per warp / CTA) */
#define EBV_BATCHED_MEDIUM_MAX_N 512  /* batched blocked schedule beyond that */

/* Column-block -> rank layouts for a 1D distribution:
 * CYCLIC = J mod P; EBVPAIR = block pairs (J, N-1-J) dealt round-robin
 * (the paper's first-with-last equalization, Eq 7, applied to blocks);
 * SNAKE = reflective (boustrophedon) order. */
typedef enum { EBV_LAYOUT_CYCLIC = 0, EBV_LAYOUT_EBVPAIR = 1, EBV_LAYOUT_SNAKE = 2 } ebv_layout_t;

/* ---- context ------------------------------------------------------------ */

/* Create a context on CUDA device `device` (made current for the call).
 * *ctx receives the handle.  Errors: INVALID_VALUE (ctx NULL, bad device),
 * CUDA, ALLOC. */
ebv_status_t ebv_create(ebv_context_t* ctx, int device);

/* Destroy a context (synchronizes the context's own resources only). */
ebv_status_t ebv_destroy(ebv_context_t ctx);

/* Static description of a status code (never NULL). */
const char* ebv_status_string(ebv_status_t s);

/* Description of the last error on the calling thread ("" if none). */
const char* ebv_last_error(void);

/* Select the factorization path (default EBV_PATH_AUTO). */
ebv_status_t ebv_set_path(ebv_context_t ctx, ebv_path_t path);

/* Blocked path leaf size (the diagonal blocks factored inside one CTA);
 * 0 restores the default.  Must be a multiple of 8 in [8, 64]. */
ebv_status_t ebv_set_leaf(ebv_context_t ctx, int64_t leaf);

/* Blocked path schedule: nb > 0 = right-looking with column blocks of nb
 * (a multiple of the leaf) — panel LU, U12 substitution, DMMA trailing
 * update per block; nb = 0 (default) = size-adaptive (64 below n = 6144, 128
 * below 12288, 256 below 24576, else 512: the best measured on B200); nb = -1 = fully
 * recursive 2 x 2 splitting.  All are bitwise identical. */
ebv_status_t ebv_set_block(ebv_context_t ctx, int64_t nb);

/* The column block width the blocked schedule will use for order n on this
 * context (the ebv_set_block value, or the size-adaptive choice; -1 for the
 * recursive schedule); 0 for a NULL ctx.  Host only, no device work. */
int64_t ebv_block_width(ebv_context_t ctx, int64_t n);

/* CUDA Graph replay of the blocked factor schedule (default on): the second
 * ebv_lu_factor call with identical arguments (same A / d_info pointers,
 * n, lda, tau and options, non-default stream) captures the schedule; later
 * calls replay it.  Bypassed while statistics are enabled. */
ebv_status_t ebv_set_graphs(ebv_context_t ctx, int enable);

/* Lookahead (default on): in the blocked schedule, panel K+1 is factored
 * on a high-priority side stream of the context while step K's update of
 * the remaining columns runs; ordering is by CUDA events, results are
 * bitwise identical either way. */
ebv_status_t ebv_set_lookahead(ebv_context_t ctx, int enable);

/* Vector path CTA count: 0 = automatic (one CTA per SM, preferring a count
 * that divides the number of column pairs); > 0 = that many CTAs with the EbV
 * paired owner map; < 0 = |ctas| CTAs with the plain cyclic map j mod C (the
 * comparison baseline for the pairing). */
ebv_status_t ebv_set_vector_ctas(ebv_context_t ctx, int64_t ctas);

/* ---- the hot path (Eq 1, Eq 6) ------------------------------------------ */

/* A = LU in place, no pivoting (Eq 6-a..c).
 *   n      order of A (n >= 0; n == 0 is a no-op that sets *d_info = 0)
 *   A      device, column-major n x n with leading dimension lda >= max(1,n);
 *          overwritten by the packed L\U factors
 *   tau    pivot floor (see the conventions above)
 *   d_info device int64: written with 0 or the first failing 1-based step
 *   stream cudaStream_t
 * Errors (synchronous, nothing launched): INVALID_VALUE for n < 0,
 * lda < max(1,n), A or d_info NULL (when n > 0), PATH_VECTOR with
 * n > EBV_VECTOR_MAX_N, or a distributed context (ebv_create_dist: use
 * ebv_lu_factor_dist; ebv_lu_solve and ebv_lu_factor_host reject it too). */
ebv_status_t ebv_lu_factor(ebv_context_t ctx, int64_t n, double* A, int64_t lda, double tau,
                           int64_t* d_info, void* stream);

/* A = LU from a HOST-resident matrix: hA (host, column-major, ldh >= n;
 * page-locked memory for full copy speed) is copied to A (device, lda >= n)
 * and factored there; A holds the packed LU (bitwise ebv_lu_factor's).
 * Default (blocked path, tau >= 0, n >= 16384): the column blocks stream in
 * on an internal copy stream and join the right-looking updates as they
 * arrive (each late block first catches up on the steps it missed, in
 * order), so most of the transfer hides under the factorization; smaller n
 * copy first on `stream`.  With EBV_PATH_LEFT (and tau >= 0) the blocks
 * stream in under the left-looking schedule.  Errors as ebv_lu_factor, plus
 * INVALID_VALUE for ldh < n or hA NULL. */
ebv_status_t ebv_lu_factor_host(ebv_context_t ctx, int64_t n, const double* hA, int64_t ldh, double* A,
                                int64_t lda, double tau, int64_t* d_info, void* stream);

/* Make `stream` wait (asynchronously) until every host-to-device transfer
 * issued by the latest ebv_lu_factor_host call on ctx has landed — e.g. to
 * start the next system's upload only after this one's, instead of sharing
 * the link with it.  No-op if no such call.  Errors: INVALID_VALUE (NULL
 * ctx), CUDA. */
ebv_status_t ebv_stream_wait_host_copy(ebv_context_t ctx, void* stream);

/* X from LY = B then UX = Y (Eq 1; "UX = B" read as UX = Y, R6).
 *   LU     device, the packed output of ebv_lu_factor (column-major, lda)
 *   B      device, n x nrhs column-major (ldb >= max(1,n)), overwritten by X
 * Each right-hand side column is processed in the canonical order (forward:
 * y_i = fma chain over ascending k of -l_ik y_k from b_i; backward: x_k =
 * y_k / u_kk, then y_i -= u_ik x_k for i < k, k descending).  A few
 * right-hand sides run as interleaved single-column wavefront chains (one
 * launch per sweep per 64 columns); many (factor once, solve many: above
 * 128, or above 64 / 40 for n > 8192 / 16384) as recursive TRSMs whose
 * off-diagonal blocks are DMMA updates — the same per-entry operations,
 * bitwise the same X.
 * Errors: INVALID_VALUE for n < 0, nrhs < 0, lda/ldb < max(1,n), NULL
 * pointers when n > 0 and nrhs > 0. */
ebv_status_t ebv_lu_solve(ebv_context_t ctx, int64_t n, const double* LU, int64_t lda, double* B,
                          int64_t ldb, int64_t nrhs, void* stream);

/* Batched independent systems (BASELINE.json configs[4]; reading R16):
 * system s has A_s = A + s*strideA (n x n column-major, lda) and, if B is not
 * NULL, right-hand sides B_s = B + s*strideB (n x nrhs, ldb), solved in place
 * (fused factor + solve).  Each system is factored exactly like
 * ebv_lu_factor (bitwise).  d_info[s] (device int32) receives each system's
 * info.  One warp holds two systems; lane t owns rows t and n-1-t of its
 * system (the paper's first-with-last pairing, Eq 7, at lane granularity).
 * Sharding across GPUs = the caller passes its shard's pointers.
 * Errors: INVALID_VALUE (n < 0, batch < 0, lda < n, strides too small,
 * NULL pointers); NOT_SUPPORTED for n > EBV_BATCHED_MEDIUM_MAX_N or
 * nrhs > 16.  Orders EBV_BATCHED_MAX_N < n <= EBV_BATCHED_MEDIUM_MAX_N (SURVEY
 * §8f f2) take the blocked schedule with 64-column steps for all systems at
 * once (every launch covers the batch): same per-system results (bitwise
 * ebv_lu_factor / the oracle). */
ebv_status_t ebv_lu_factor_batched(ebv_context_t ctx, int64_t n, double* A, int64_t lda,
                                   int64_t strideA, int64_t batch, double* B, int64_t ldb,
                                   int64_t strideB, int64_t nrhs, double tau, int32_t* d_info,
                                   void* stream);

/* Banded / sparse inputs (the paper's second workload, P:93-103, P:119;
 * SURVEY §8f f4): A (dense column-major storage, lda >= n) has a_ij = 0 for
 * i - j > kl and j - i > ku.  No-pivot LU keeps that band (L lower bandwidth
 * kl, U upper bandwidth ku), so the blocked schedule clips every panel, U12
 * and DMMA update to it (zero-skip: work ~ n*kl*ku instead of n^3); entries
 * outside the band are not touched.  The factors are bitwise ebv_lu_factor's
 * (the skipped operations are exact no-ops on zeros) for inputs with positive
 * pivots (a negative pivot would give -0 instead of +0 below the band in the
 * dense algorithm).  ebv_lu_solve_banded skips the zero tiles of the
 * substitutions.  Errors as ebv_lu_factor / ebv_lu_solve, plus
 * INVALID_VALUE for kl < 0 or ku < 0. */
ebv_status_t ebv_lu_factor_banded(ebv_context_t ctx, int64_t n, int64_t kl, int64_t ku, double* A,
                                  int64_t lda, double tau, int64_t* d_info, void* stream);
ebv_status_t ebv_lu_solve_banded(ebv_context_t ctx, int64_t n, int64_t kl, int64_t ku, const double* LU,
                                 int64_t lda, double* B, int64_t ldb, int64_t nrhs, void* stream);

/* Banded systems in compact band storage (memory
 * ~ n*(kl+ku) instead of n^2, so orders far beyond the dense limit fit).
 * AB is ldab x n column-major (device, caller-owned); entry a_ij of the band
 * (max(0, j-ku) <= i <= min(n-1, j+kl)) lives at
 *     AB[(EBV_BAND_PAD + ku + i - j) + j*ldab],
 * i.e. LAPACK's band layout with EBV_BAND_PAD extra rows above and below:
 * the blocked schedule works on 64-column steps whose panels, U12 blocks and
 * solve tiles reach up to EBV_BAND_PAD entries past the band (exact zeros).
 * Requires ldab >= kl + ku + 2*EBV_BAND_PAD + 1 and every entry of AB outside
 * the band zero on entry.  The factor overwrites the band with L\U in the
 * same layout (padding entries may become +-0); the factors in the band are
 * bitwise ebv_lu_factor_banded's on the same matrix in dense storage.  The
 * pivot threshold must be explicit (tau >= 0: the tau < 0 norm rule needs
 * the dense layout).  The solve (Eq 1) overwrites B (n x nrhs, ldb) with X.
 * Errors: INVALID_VALUE (negative sizes, ldab too small, tau < 0, NULL
 * pointers), plus the conditions of ebv_lu_factor / ebv_lu_solve. */
#define EBV_BAND_PAD 128
ebv_status_t ebv_lu_factor_band(ebv_context_t ctx, int64_t n, int64_t kl, int64_t ku, double* AB,
                                int64_t ldab, double tau, int64_t* d_info, void* stream);
ebv_status_t ebv_lu_solve_band(ebv_context_t ctx, int64_t n, int64_t kl, int64_t ku, const double* AB,
                               int64_t ldab, double* B, int64_t ldb, int64_t nrhs, void* stream);

/* Solve only, for batched systems factored earlier by ebv_lu_factor_batched
 * (factor once, solve many — SURVEY §8f f1): for each system s,
 * B_s <- U_s^-1 (L_s^-1 B_s) with the packed LU_s = LU + s*strideA (read
 * only), forward then backward substitution of Eq 1 per column in
 * the canonical order (bitwise ebv_lu_solve / the oracle on each system).
 * Layout, strides and limits as ebv_lu_factor_batched (n <= 512,
 * nrhs <= 16).  Errors: INVALID_VALUE, NOT_SUPPORTED as there. */
ebv_status_t ebv_lu_solve_batched(ebv_context_t ctx, int64_t n, const double* LU, int64_t lda,
                                  int64_t strideA, int64_t batch, double* B, int64_t ldb,
                                  int64_t strideB, int64_t nrhs, void* stream);

/* Unit-diagonal normalization (Eq 2: the coefficient matrix drawn
 * with 1 on its diagonal): row i of A (n x n,
 * lda) and, if B != NULL, of B (n x nrhs, ldb) divided by a_ii — one
 * correctly rounded division per entry, so the diagonal becomes exactly 1
 * and the solution is unchanged up to rounding; d_scales[i] = 1/a_ii (may be
 * NULL).  A row with a_ii == 0 is left unchanged (scale 0) and reported in
 * d_info (device int64) as the first such 1-based row, else 0.  All pointers
 * device, column-major; asynchronous on `stream`.
 * Errors: INVALID_VALUE for negative sizes, leading dimensions < n, NULL
 * A / d_info. */
ebv_status_t ebv_normalize_unit_diagonal(ebv_context_t ctx, int64_t n, double* A, int64_t lda, double* B,
                                         int64_t ldb, int64_t nrhs, double* d_scales, int64_t* d_info,
                                         void* stream);

/* LDU form of a packed LU from ebv_lu_factor (Eq 3, which draws U
 * with a unit diagonal; Eq 6-b's U_(k) row divided by its pivot):
 * A = L D U' with D = diag(U) copied to d_D (device, n doubles) and, in
 * place, u'_kj = u_kj / u_kk for j > k (one correctly rounded division); the
 * strict lower triangle (L) and the diagonal (D) are unchanged, U' has an
 * implicit unit diagonal.  Errors: INVALID_VALUE for n < 0, lda < n, NULL
 * pointers. */
ebv_status_t ebv_lu_to_ldu(ebv_context_t ctx, int64_t n, double* LU, int64_t lda, double* d_D, void* stream);

/* The trailing rank-k update of Eq 6-c on its own — the DMMA
 * contraction every blocked / distributed schedule is built from:
 *     C <- C - A * B      A: M x K (lda), B: K x N (ldb), C: M x N (ldc),
 * all device, column-major.  Each entry of C is the fma chain
 * c <- fma(-a_ik, b_kj, c) over k = 0..K-1 ascending starting from its input
 * value (bitwise the oracle's order for those k).  Errors: INVALID_VALUE for
 * negative sizes, leading dimensions below the row counts, NULL pointers
 * when the product is non-empty. */
ebv_status_t ebv_update(ebv_context_t ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                        const double* B, int64_t ldb, double* C, int64_t ldc, void* stream);

/* ---- multi-GPU: batched systems (C5) sharded over P GPUs --- */
/* Contiguous, balanced system range of `rank` among `nranks` (host only):
 * ranks < batch % nranks take one extra system.  Each rank then calls
 * ebv_lu_factor_batched on its range — no collective on the data path.
 * Errors: INVALID_VALUE for batch < 0, nranks < 1, rank out of range, NULL
 * outputs. */
ebv_status_t ebv_batched_shard(int64_t batch, int rank, int nranks, int64_t* first, int64_t* count);

/* ---- multi-GPU: one system over P GPUs -------- */
/* 1D block-cyclic columns: column block J (width nb, the last one ragged)
 * lives on rank ebv_block_owner(J, N, P, layout); a rank stores its blocks
 * in ascending J as a column-major n x local_cols slab (ld >= n).  Per step K
 * the owner factors the panel and broadcasts it over NCCL (in place, on the
 * caller's stream); every rank substitutes and updates its blocks J > K.
 * For a fixed nb the results are bitwise identical for every P and equal to
 * ebv_lu_factor with ebv_set_block(nb) (and to the serial oracle).
 * NCCL is loaded at run time (libnccl.so.2; EBV_NCCL_LIB overrides the
 * path); all ranks must make the same calls in the same order. */

/* 128-byte NCCL unique id for ebv_create_dist (call on one rank, share the
 * bytes with the others, e.g. through torch.distributed).  Errors: NCCL. */
ebv_status_t ebv_get_unique_id(void* uid);

/* Context for rank `rank` of `nranks` on `device`, with its own NCCL
 * communicator; nb: column block width (positive multiple of 64).
 * Collective: every rank must call it.  Errors: INVALID_VALUE, NCCL, CUDA. */
ebv_status_t ebv_create_dist(ebv_context_t* ctx, int device, const void* uid, int rank, int nranks, int64_t nb,
                             ebv_layout_t layout);

/* Number of ranks in the context's NCCL communicator (ncclCommCount; the
 * nranks given to ebv_create_dist if NCCL cannot report it); -1 for a NULL
 * or non-distributed context. */
int ebv_dist_nranks(ebv_context_t ctx);

/* Host, pure: the column blocks rank `rank` owns (ascending J; blocks may be
 * NULL to query the count), their count and the slab width local_cols. */
ebv_status_t ebv_dist_local_blocks(int64_t n, int64_t nb, int rank, int nranks, ebv_layout_t layout, int64_t* blocks,
                                   int64_t cap, int64_t* nblocks, int64_t* local_cols);

/* Distributed A = LU (Eq 6): A_local is this rank's slab (device, column-
 * major, lda >= n), factored in place; d_info (device int64) receives the
 * global first failing step on every rank.  tau < 0 selects the default
 * floor n*eps*||A||_inf from the global row sums (each rank's partial row
 * sums added by an NCCL all-reduce: bitwise the single-GPU floor when the
 * row sums are exact, else equal up to the summation order, reading R18).
 * Collective. */
ebv_status_t ebv_lu_factor_dist(ebv_context_t ctx, int64_t n, double* A_local, int64_t lda, double tau,
                                int64_t* d_info, void* stream);

/* Distributed solve (Eq 1) with the factors of ebv_lu_factor_dist: B (device,
 * n x nrhs, ldb >= n) holds the same right-hand sides on every rank and is
 * overwritten with X on every rank.  Forward / backward substitution pass B
 * through the block owners in order (ncclSend / ncclRecv), so every entry is
 * computed in the canonical order.  Collective. */
ebv_status_t ebv_lu_solve_dist(ebv_context_t ctx, int64_t n, const double* LU_local, int64_t lda, double* B,
                               int64_t ldb, int64_t nrhs, void* stream);

/* Single-GPU emulation of the P-rank schedule (validation on one device):
 * slabs is a HOST array of nranks device pointers, slab r laid out exactly as
 * rank r's A_local; ctx is an ordinary context.  Same results as the real
 * distributed calls. */
ebv_status_t ebv_lu_factor_dist_emulated(ebv_context_t ctx, int64_t n, int nranks, int64_t nb, ebv_layout_t layout,
                                         double* const* slabs, int64_t lda, double tau, int64_t* d_info,
                                         void* stream);
ebv_status_t ebv_lu_solve_dist_emulated(ebv_context_t ctx, int64_t n, int nranks, int64_t nb, ebv_layout_t layout,
                                        double* const* slabs, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                                        void* stream);

/* ---- EbV plan (host, pure; Eq 7) -------------------------- */

/* Owner map over n indices (columns, rows or blocks): index j is paired with
 * n-1-j (first with last), pairs p = 0,1,... dealt round-robin to `workers`
 * (reading R12).  owner: host array of n int32.  Errors: INVALID_VALUE. */
ebv_status_t ebv_plan_owner_map(int64_t n, int64_t workers, int32_t* owner);

/* The paper's equal-length units (Eq 7; SPEC equalize): for n >= 2 exactly
 * n-1 units.  Unit u is written as (tri0[u], k0[u], tri1[u], k1[u]) with
 * tri = 0 for an L vector, 1 for a U vector, k 1-based, and tri1 = -1 for a
 * single-member unit (never produced: every unit has two members), plus its
 * round-robin owner.  Arrays have n-1 entries.  Errors: INVALID_VALUE. */
ebv_status_t ebv_plan_units(int64_t n, int64_t workers, int32_t* tri0, int32_t* k0, int32_t* tri1,
                            int32_t* k1, int32_t* owner);

/* Owner rank of column block J of N blocks over nranks under `layout`
 * (-1 on invalid arguments). */
int64_t ebv_block_owner(int64_t J, int64_t N, int64_t nranks, ebv_layout_t layout);

/* ---- debug knobs (validation; process-wide per device) -------------------- */
/* flags:
 *   EBV_DEBUG_FORCE_EXACT  every verified-quotient test (the Markstein
 *       quotient from a hoisted reciprocal used on the division chains of
 *       the solve, leaf, vector and batched kernels) reports "unverified", so
 *       every such step takes its redo-with-true-division branch.  Results
 *       must not change (they are RN(y/u) either way); slower.
 *   EBV_DEBUG_JITTER  pseudo-random sleeps (0..4 us) before cross-CTA flag
 *       releases, to stress the flag protocols' ordering.
 * spin_timeout_s: bound on any one cross-CTA flag wait; a wait that exceeds
 * it traps (the launch fails with a CUDA error instead of hanging the GPU).
 * 0 = unbounded; the default is 60 s.  Applies to kernels launched on
 * `device` after the call.  Errors: INVALID_VALUE (unknown flag, bad device,
 * timeout < 0), CUDA. */
#define EBV_DEBUG_FORCE_EXACT 1u
#define EBV_DEBUG_JITTER 2u
ebv_status_t ebv_set_debug(int device, unsigned flags, double spin_timeout_s);

/* ---- measurement --------------------------------------------------------- */

/* Per-kernel-class statistics, recorded with CUDA events on the launching
 * stream while enabled (off by default).  Classes: 0 = other DMMA launches
 * (inside the recursive TRSMs and panels), 1 = diagonal-block LU (panel
 * leaves), 2 = TRSM, 3 = solve, 4 = batched, 5 = vector path, 6 = other,
 * 7 = the trailing rank-nb update of Eq 6-c (DMMA; the dominant kernel).  ebv_stats_get synchronizes the events and
 * returns for class c: launches, total milliseconds, algorithmic flops and
 * algorithmic bytes. */
#define EBV_NUM_KCLASSES 8
ebv_status_t ebv_stats_enable(ebv_context_t ctx, int enable);
ebv_status_t ebv_stats_reset(ebv_context_t ctx);
ebv_status_t ebv_stats_get(ebv_context_t ctx, int kclass, int64_t* launches, double* ms,
                           double* flops, double* bytes);

/* The recorded launches since the last reset as a timeline: writes up to
 * max_records triples (class, start ms, end ms) to out (class + 256 when
 * the launch went to the lookahead side stream), times relative to
 * the first recorded launch's start, in launch order; returns the number of
 * records available (-1 on invalid arguments).  Synchronizes like
 * ebv_stats_get.  A diagnostic: the bracketing events add a little time. */
int64_t ebv_stats_timeline(ebv_context_t ctx, double* out, int64_t max_records);

/* Number of kernels this context launched since creation (all classes). */
int64_t ebv_launch_count(ebv_context_t ctx);

#ifdef __cplusplus
}
#endif
#endif /* EBV_H_ */
