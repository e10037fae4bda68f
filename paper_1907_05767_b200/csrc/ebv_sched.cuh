// ebv_sched.cuh — the context object and the schedule helpers shared by the
// host translation units (ebv_api.cu: single-GPU schedules and the C ABI;
// ebv_dist.cu: the 1D block-cyclic multi-GPU schedule).  Internal.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "ebv_internal.cuh"

struct ebv_dist_state;   // ebv_dist.cu

struct ebv_context {
  int device = 0;
  ebv_path_t path = EBV_PATH_AUTO;
  int64_t leaf = 64;
  int64_t nb = 0;           // right-looking block width; 0 = size-adaptive, -1 = fully recursive
  double* d_tau = nullptr;
  unsigned long long* d_norm = nullptr;
  double* d_scratch = nullptr;
  int* d_ticket = nullptr;
  int* d_pcount = nullptr;
  double* d_vec = nullptr;  // n-vector workspace (row scalings)
  void* d_bws = nullptr;    // batched medium path: per-system tau, info, arrival counters
  int64_t bws_cap = 0;
  int64_t vec_cap = 0;  // panel-leaf arrival counter (zero between launches; self-resetting)
  int* d_flags = nullptr;
  int64_t flags_cap = 0;
  int* d_vflags = nullptr;
  int64_t vflags_cap = 0;
  int64_t solve_epoch = 0;  // flag epochs consumed by the wavefront solves (d_flags)
  int64_t vector_epoch = 0; // flag epochs consumed by the vector path (d_vflags)
  int64_t launches = 0;
  int vector_ctas = 0;      // 0 = auto; < 0 = cyclic map with |value| CTAs (for comparison)
  bool lookahead = true;    // factor panel K+1 on a side stream under the update of step K
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_a = nullptr, ev_p = nullptr, ev_b = nullptr;
  cudaStream_t copy = nullptr;            // host -> device column blocks (ebv_lu_factor_host)
  std::vector<cudaEvent_t> copy_ev;       // one per column block
  cudaEvent_t hostcopy_ev = nullptr;      // after the last host copy of the last ebv_lu_factor_host
  bool hostcopy_valid = false;
  bool stats = false;
  struct Rec {
    int cls;
    cudaEvent_t e0, e1;
    double flops, bytes;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  int64_t st_launch[EBV_NUM_KCLASSES] = {0};
  double st_ms[EBV_NUM_KCLASSES] = {0}, st_flops[EBV_NUM_KCLASSES] = {0}, st_bytes[EBV_NUM_KCLASSES] = {0};
  std::vector<double> tl;           // stats timeline: (class, start ms, end ms) per launch
  cudaEvent_t tl_ref = nullptr;     // the timeline's time origin (first launch since reset)
  ebv_dist_state* dist = nullptr;   // set by ebv_create_dist
  // CUDA Graph cache of the blocked factor schedule, keyed by its arguments
  bool graphs = true;
  struct GraphEntry {
    int64_t n, lda, nb, leaf;
    const void* A;
    const void* info;
    double tau;
    bool la;
    int hits;
    int64_t launches;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> gcache;
};


namespace ebv {
namespace sched {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

ebv_status_t cuda_fail(cudaError_t e, const char* where);
ebv_status_t invalid(const char* msg);
cudaEvent_t get_event(ebv_context* c);

// Launch wrapper: counts launches and (when enabled) brackets the launch with
// CUDA events on the launching stream for the per-class statistics.
template <class F>
cudaError_t timed(ebv_context* c, int cls, double flops, double bytes, cudaStream_t s, int nlaunch, F&& f) {
  c->launches += nlaunch;
  if (!c->stats) return f();
  ebv_context::Rec r{cls | (s != nullptr && s == c->side ? 256 : 0), get_event(c), get_event(c), flops, bytes};
  cudaEventRecord(r.e0, s);
  cudaError_t e = f();
  cudaEventRecord(r.e1, s);
  c->recs.push_back(r);
  return e;
}

cudaError_t gemm(ebv_context* c, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                 int64_t ldb, double* C, int64_t ldc, bool rev, cudaStream_t s, int cls = KC_GEMM);
int64_t split_point(int64_t n, int64_t leaf);
cudaError_t trsm_r(ebv_context* c, int64_t m, int64_t k, double* X, int64_t ldx, const double* U, int64_t ldu,
                   cudaStream_t s);
cudaError_t trsm_l(ebv_context* c, int64_t k, int64_t m, const double* L, int64_t ldl, double* X, int64_t ldx,
                   cudaStream_t s);
cudaError_t trsm_lu(ebv_context* c, int64_t k, int64_t m, const double* U, int64_t ldu, double* X, int64_t ldx,
                    cudaStream_t s);
cudaError_t lu_rec(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t koff, int64_t* info, cudaStream_t s);
cudaError_t panel_rec(ebv_context* c, int64_t M, int64_t w, double* P, int64_t lda, int64_t koff, int64_t* info,
                      cudaStream_t s);
cudaError_t lu_blocked(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t* info, cudaStream_t s,
                       int64_t kl, int64_t ku, bool band_storage = false);
cudaError_t lu_left(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t* info, cudaStream_t s,
                    const double* hA, int64_t ldh);
cudaError_t lu_blocked_stream(ebv_context* c, int64_t n, double* A, int64_t lda, int64_t* info, cudaStream_t s,
                              const double* hA, int64_t ldh);
void dist_release(ebv_context* c);   // ebv_dist.cu
// the single-GPU solve (chain / wavefront / TRSM by shape), ebv_api.cu
ebv_status_t solve_full(ebv_context* c, int64_t n, const double* LU, int64_t lda, double* B, int64_t ldb,
                        int64_t nrhs, cudaStream_t s);

}  // namespace sched
}  // namespace ebv
