// ebv_internal.cuh — internal declarations shared by the libebv translation
// units (kernels + host dispatch).  Not part of the public C ABI (include/ebv.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/ebv.h"

namespace ebv {

// Kernel classes for the measurement hooks (ebv_stats_*).
enum KClass { KC_GEMM = 0, KC_LEAF = 1, KC_TRSM = 2, KC_SOLVE = 3, KC_BATCHED = 4, KC_VECTOR = 5,
              KC_OTHER = 6, KC_UPDATE = 7 };

void set_error(const std::string& msg);

// ---- launchers (all asynchronous on `s`; return cudaGetLastError()) -------

// C <- C - A*B  (A: M x K col-major lda, B: K x N col-major ldb, C: M x N ldc).
// Every entry of C is the fma chain c <- fma(-a_ik, b_kj, c) over k ascending
// (or descending when reverse_k), starting from its input value: the FP64
// tensor-core (DMMA) contraction of the Eq 6-c rank-k update.
cudaError_t launch_gemm_sub(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                            const double* B, int64_t ldb, double* C, int64_t ldc, bool reverse_k,
                            cudaStream_t s);

// TMA-fed variant (k_gemm_tma.cu); eligible for 16-byte aligned bases and
// even leading dimensions.
bool gemm_tma_eligible(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B, int64_t ldb);
cudaError_t launch_gemm_sub_tma(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                                int64_t ldb, double* C, int64_t ldc, int variant, cudaStream_t s);

// 2-D TMA descriptor (CUtensorMap, 128 bytes at `map`) of a column-major
// fp64 matrix rows x cols with leading dimension ld and box box0 x box1
// (out-of-range elements read as zero); false if the driver cannot make it.
bool make_tma_map_2d(void* map, const double* ptr, int64_t rows, int64_t cols, int64_t ld, int box0, int box1);

// Unblocked LU of one diagonal block (n <= 64) inside one CTA (Eq 6-a..c).
// Pivot check against *tau (device); the first failing step (1-based,
// global index koff + k + 1) is written to *info if *info is still 0.
cudaError_t launch_leaf_lu(int64_t n, double* A, int64_t lda, const double* tau, int64_t* info,
                           int64_t koff, cudaStream_t s);

// X <- X U^-1, U upper triangular k x k (k <= 64, non-unit), X m x k:
// row-parallel substitution (the L21 panel of the blocked form).
// Batched forms of the blocked-schedule kernels (systems at base + s*stride,
// s < batch): per system bitwise the single-system launches.  Used by the
// batched medium-order path (ebv_lu_factor_batched, 64 < n <= 512).
cudaError_t launch_panel_leaf_batched(int64_t M, int64_t w, double* P, int64_t lda, int64_t bsP, const double* tau,
                                      int64_t bsTau, int64_t* info, int64_t bsInfo, int64_t koff, int* count,
                                      int64_t batch, cudaStream_t s);
cudaError_t launch_trsm_llu_batched(int64_t k, int64_t m, const double* L, int64_t ldl, int64_t bsL, double* X,
                                    int64_t ldx, int64_t bsX, int64_t batch, cudaStream_t s);
cudaError_t launch_trsm_luu_batched(int64_t k, int64_t m, const double* U, int64_t ldu, int64_t bsU, double* X,
                                    int64_t ldx, int64_t bsX, int64_t batch, cudaStream_t s);
cudaError_t launch_gemm_sub_batched(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int64_t sA,
                                    const double* B, int64_t ldb, int64_t sB, double* Cm, int64_t ldc, int64_t sC,
                                    int64_t batch, bool reverse_k, cudaStream_t s);

cudaError_t launch_panel_leaf(int64_t M, int64_t w, double* P, int64_t lda, const double* tau, int64_t* info,
                              int64_t koff, int* count, cudaStream_t s);
cudaError_t launch_trsm_right_upper(int64_t m, int64_t k, double* X, int64_t ldx, const double* U,
                                    int64_t ldu, cudaStream_t s);

// X <- L^-1 X, L unit lower triangular k x k (k <= 64), X k x m:
// column-parallel substitution (the U12 panel of the blocked form).
cudaError_t launch_trsm_left_lower_unit(int64_t k, int64_t m, const double* L, int64_t ldl, double* X,
                                        int64_t ldx, cudaStream_t s);

// X <- U^-1 X, U upper triangular non-unit k x k (k <= 64), X k x m:
// column-parallel backward substitution, k descending.
cudaError_t launch_trsm_left_upper(int64_t k, int64_t m, const double* U, int64_t ldu, double* X, int64_t ldx,
                                   cudaStream_t s);

// Forward (LY = B) then backward (UX = Y) wavefront substitution (Eq 1).
cudaError_t launch_solve_window(int64_t n, const double* LUw, int64_t ldl, int64_t c0, int64_t w, bool fwd, double* B,
                                int64_t ldb, int64_t nrhs, int* ticket, int* flags, int epoch, cudaStream_t s);
int64_t solve_max_rhs();

// Row scalings (k_scale.cu).  dws: n doubles of workspace.
cudaError_t launch_normalize_unit_diagonal(int64_t n, double* A, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                                           double* scales, int64_t* info, double* dws, unsigned long long* info_min,
                                           cudaStream_t s, int64_t* launches);
cudaError_t launch_lu_to_ldu(int64_t n, double* LU, int64_t lda, double* D, cudaStream_t s, int64_t* launches);
int64_t solve_max_interleave();
cudaError_t launch_solve(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                         int* ticket_ws, int* flags_ws, int64_t epoch, cudaStream_t s,
                         int64_t kl = -1, int64_t ku = -1);
int64_t solve_block_rows();
// Chain-pipelined solve (k_solve2.cu): eligibility, flag ints per sweep
// (two sweeps: 2x), epochs consumed per call.
bool solve_chain_eligible(int64_t n, const double* LU, int64_t lda, int64_t nrhs);
int64_t solve_chain_flags(int64_t n);
int64_t solve_chain_epochs(int64_t nrhs);
cudaError_t launch_solve_chain(int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                               int* flags_ws, int64_t epoch, cudaStream_t s);

// flag epochs one launch_solve call consumes (base + 1 .. base + this)
int64_t launch_solve_epochs(int64_t nrhs);

// Batched n <= 32 fused factor + solve.
cudaError_t launch_batched(int64_t n, double* A, int64_t lda, int64_t strideA, int64_t batch, double* B,
                           int64_t ldb, int64_t strideB, int64_t nrhs, const double* tau, bool tau_default,
                           double tau_value, int32_t* info, cudaStream_t s,
                           bool solve_only = false);

// Vector-level EbV path (persistent cooperative kernel).
cudaError_t launch_vector_lu(int64_t n, double* A, int64_t lda, const double* tau, int64_t* info,
                             int* flags_ws, double* lbuf_ws, int num_ctas, int epoch, cudaStream_t s);
int vector_max_ctas(int device, int64_t n);
size_t vector_smem_bytes(int64_t n, int num_ctas);

// Debug knobs (ebv_set_debug): each kernel translation unit's setter of its
// __constant__ copy (ebv_device.cuh, EBV_DEBUG_SETTER).
struct DebugCfg;
cudaError_t set_debug_solve(const DebugCfg& cfg);
cudaError_t set_debug_vector(const DebugCfg& cfg);
cudaError_t set_debug_batched(const DebugCfg& cfg);
cudaError_t set_debug_leaf(const DebugCfg& cfg);
cudaError_t set_debug_solve_chain(const DebugCfg& cfg);

// Utilities.
cudaError_t launch_set_info0(int64_t* info, cudaStream_t s);
// cudaFuncSetAttribute(fn, MaxDynamicSharedMemorySize, bytes) once per
// (kernel, device) — the attribute is per device, so a process that drives
// several GPUs sets it on each (thread-safe).
cudaError_t ensure_max_dyn_smem(const void* fn, int bytes);
// batched medium path: per-system pivot floors and cleared int64 info words;
// int64 info words -> the API's int32 per-system info
cudaError_t launch_batched_prep(int64_t n, const double* A, int64_t lda, int64_t sA, int64_t batch, double tau,
                                double* tau_s, int64_t* info64, cudaStream_t s);
cudaError_t launch_info_to_i32(int64_t batch, const int64_t* info64, int32_t* info32, cudaStream_t s);
// distributed default floor: rs[i] (+)= sum_j |A[i + j*lda]| over cols
// local columns (j ascending; first: rs overwritten), then
// tau_out = n * eps * max_i rs[i]
cudaError_t launch_rowabs(int64_t n, const double* A, int64_t lda, int64_t cols, double* rs, bool first,
                          cudaStream_t s);
cudaError_t launch_tau_from_rows(int64_t n, const double* rs, double* tau_out, cudaStream_t s);
// tau_out = (tau >= 0) ? tau : n * eps * ||A||_inf  (norm pre-pass)
cudaError_t launch_tau(int64_t n, const double* A, int64_t lda, double tau, double* tau_out,
                       unsigned long long* norm_ws, cudaStream_t s);

}  // namespace ebv
