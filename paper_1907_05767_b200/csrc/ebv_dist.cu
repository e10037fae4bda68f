// ebv_dist.cu — the multi-GPU schedule: one large
// system factored over P GPUs with a 1D block-cyclic column layout and an
// NCCL broadcast of each factored panel over NVLink / NVSwitch; the solve is
// a ring that carries the right-hand side through the block owners in order.
//
// Paper: the method is "convenient for ... multi devices"; the
// per-step structure is Eq 6 in block form.  For a fixed block
// width nb every entry sees exactly the operation sequence of the one-GPU
// blocked schedule (panel LU, U12 substitution, DMMA update with k ascending),
// so the factors and the solution are bitwise identical for every P and
// equal to the serial oracle.
//
// Step K (owner = ebv_block_owner(K, N, P, layout)):
//   owner   : panel LU of its block K (rows K*nb..n) in place, pack the panel
//             (L11\U11 over L21, contiguous M x w) into the panel buffer
//   all     : ncclBroadcast of the panel buffer from the owner (in place)
//   all     : U12 = L11^-1 A12 and A22 -= L21 U12 on their local blocks J > K
//             (a contiguous suffix of the local slab: blocks are stored in
//             ascending J)
// Solve, forward (K ascending) then backward (K descending): owner(K) solves
// its diagonal block against the current right-hand side, applies its block
// column to the rows below (above, with the reverse-k update), and passes
// the right-hand side to owner(K+1) (owner(K-1)) with ncclSend / ncclRecv;
// the result is broadcast from owner(0).
//
// The same driver runs in an emulation mode: one process, one GPU, all P
// virtual ranks' slabs; the "broadcast" is the shared panel buffer and the
// ring is the shared right-hand side.  It validates the multi-rank schedule
// (ownership, local offsets, packing) bitwise on a single GPU.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, the copy torch ships),
// so libebv.so has no link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <climits>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "ebv_sched.cuh"

using namespace ebv;
using namespace ebv::sched;

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclBroadcast) Broadcast = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclCommCount) CommCount = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = getenv("EBV_NCCL_LIB");
    void* h = nullptr;
    if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define EBV_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    EBV_SYM(GetUniqueId);
    EBV_SYM(CommInitRank);
    EBV_SYM(CommDestroy);
    EBV_SYM(Broadcast);
    EBV_SYM(AllReduce);
    EBV_SYM(Send);
    EBV_SYM(Recv);
    EBV_SYM(GetErrorString);
    EBV_SYM(CommCount);
#undef EBV_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Broadcast && api.AllReduce &&
             api.Send && api.Recv;
  });
  return api;
}

// EBV_DIST_FORCE_NCCL=1: a one-rank communicator still takes the NCCL data
// path (panel broadcasts, info / row-sum all-reduces, the ring solve and its
// final broadcast) — a one-rank collective is a local copy, so the calls,
// their streams and the event protocol around them run on one GPU (tests)
bool force_nccl() {
  static const bool v = [] {
    const char* e = getenv("EBV_DIST_FORCE_NCCL");
    return e && atoi(e) == 1;
  }();
  return v;
}

ebv_status_t nccl_fail(ncclResult_t r, const char* where) {
  const char* m = nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error";
  set_error(std::string(where) + ": " + m);
  return EBV_ERR_NCCL;
}

// local column blocks of `rank` in ascending J, their slab offsets and widths
struct Plan {
  int64_t n = 0, nb = 0, N = 0;
  int P = 1, rank = 0;
  ebv_layout_t layout = EBV_LAYOUT_CYCLIC;
  std::vector<int64_t> blocks, off;   // local block list and local column offsets
  std::vector<int64_t> loc;           // global J -> local offset or -1
  int64_t cols = 0;
  int64_t width(int64_t J) const { return (J + 1) * nb <= n ? nb : n - J * nb; }
  int64_t owner(int64_t J) const { return ebv_block_owner(J, N, P, layout); }
};

Plan make_plan(int64_t n, int64_t nb, int rank, int P, ebv_layout_t layout) {
  Plan p;
  p.n = n; p.nb = nb; p.P = P; p.rank = rank; p.layout = layout;
  p.N = (n + nb - 1) / nb;
  p.loc.assign(p.N, -1);
  for (int64_t J = 0; J < p.N; J++)
    if (p.owner(J) == rank) {
      p.blocks.push_back(J);
      p.off.push_back(p.cols);
      p.loc[J] = p.cols;
      p.cols += p.width(J);
    }
  return p;
}

// first local column of a block J' > K, or cols
int64_t suffix_after(const Plan& p, int64_t K) {
  for (size_t b = 0; b < p.blocks.size(); b++)
    if (p.blocks[b] > K) return p.off[b];
  return p.cols;
}

struct View {
  Plan plan;
  double* A;
  int64_t lda;
};

__global__ void info_to_min_kernel(int64_t* info) {
  if (*info == 0) *info = INT64_MAX;
}
__global__ void info_from_min_kernel(int64_t* info) {
  if (*info == INT64_MAX) *info = 0;
}

}  // namespace

struct ebv_dist_state {
  int rank = 0, nranks = 1;
  int64_t nb = 256;
  ebv_layout_t layout = EBV_LAYOUT_CYCLIC;
  ncclComm_t comm = nullptr;
  double* pbuf = nullptr;       // two panel buffers (double-buffered), each pcap/2
  size_t pcap = 0;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr};   // panel K broadcast complete (side)
  cudaEvent_t ev_free[2] = {nullptr, nullptr};    // step K done reading pbuf[K%2] (main)
  cudaEvent_t ev_next = nullptr;                  // block K+1 columns updated (main)
  cudaEvent_t ev_brow = nullptr;                  // block row K+1 of the local columns updated (main)
  cudaEvent_t ev_side = nullptr;                  // join point of the side stream
  int* sws = nullptr;           // ring-solve workspace: per RHS group, the two sweeps' row-block
  int64_t sws_cap = 0;          // flags, then one launch ticket per (window, sweep, group)
};

namespace {

ebv_status_t ensure_pbuf(ebv_context* c, ebv_dist_state* d, size_t elems) {
  if (!d->ev_next) {
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; i++) {
      e = cudaEventCreateWithFlags(&d->ev_ready[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_free[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_next, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_brow, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_side, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "dist events");
  }
  if (2 * elems <= d->pcap) return EBV_SUCCESS;
  if (d->pbuf) cudaFree(d->pbuf);
  d->pbuf = nullptr;
  d->pcap = 0;
  cudaError_t e = cudaMalloc(&d->pbuf, 2 * elems * sizeof(double));
  if (e != cudaSuccess) { set_error("panel buffer alloc failed"); return EBV_ERR_ALLOC; }
  d->pcap = 2 * elems;
  (void)c;
  return EBV_SUCCESS;
}

void release_events(ebv_dist_state* d) {
  for (int i = 0; i < 2; i++) {
    if (d->ev_ready[i]) cudaEventDestroy(d->ev_ready[i]);
    if (d->ev_free[i]) cudaEventDestroy(d->ev_free[i]);
  }
  if (d->ev_next) cudaEventDestroy(d->ev_next);
  if (d->ev_brow) cudaEventDestroy(d->ev_brow);
  if (d->ev_side) cudaEventDestroy(d->ev_side);
}

// The schedule over the views this process drives (one real rank, or all P
// virtual ranks in emulation).  comm == nullptr means emulation.
//
// Streams: every panel factorization, pack and broadcast runs on the side
// stream (one NCCL stream, collectives in step order on every rank); the
// updates run on the caller's stream.  Lookahead: at step K the owner of
// block K+1 updates those columns first, then factors panel K+1 on the side
// stream while its caller stream updates the rest of its slab, so panel
// K+1 (and its broadcast) overlaps step K's updates.  Panel buffers are
// double-buffered by step parity; events order the reuse.
ebv_status_t dist_factor(ebv_context* c, ebv_dist_state* d, std::vector<View>& views, int64_t n, int64_t* info,
                         cudaStream_t s) {
  const Plan& p0 = views[0].plan;
  const int64_t nb = p0.nb, N = p0.N;
  const size_t half = (size_t)n * nb;
  ebv_status_t st = ensure_pbuf(c, d, half);
  if (st != EBV_SUCCESS) return st;
  const bool real = d->comm && (d->nranks > 1 || force_nccl());
  cudaStream_t side = c->side;
  cudaError_t e = cudaEventRecord(d->ev_side, s);                  // side starts after the caller's work
  if (e == cudaSuccess) e = cudaStreamWaitEvent(side, d->ev_side, 0);
  if (e != cudaSuccess) return cuda_fail(e, "dist fork");
  auto pbuf = [&](int64_t K) { return d->pbuf + (size_t)(K & 1) * half; };

  // factor + pack panel K (owner's view) on the side stream
  auto prepare_panel = [&](int64_t K) -> cudaError_t {
    const int64_t c0 = K * nb, w = p0.width(K), M = n - c0;
    for (auto& v : views) {
      if (v.plan.rank != p0.owner(K)) continue;
      double* P = v.A + c0 + v.plan.loc[K] * v.lda;
      cudaError_t e2 = panel_rec(c, M, w, P, v.lda, c0, info, side);
      if (e2 != cudaSuccess) return e2;
      if (K >= 2) {   // pbuf[K%2] was read by step K-2 on the caller stream
        e2 = cudaStreamWaitEvent(side, d->ev_free[K & 1], 0);
        if (e2 != cudaSuccess) return e2;
      }
      e2 = cudaMemcpy2DAsync(pbuf(K), M * sizeof(double), P, v.lda * sizeof(double), M * sizeof(double), w,
                             cudaMemcpyDeviceToDevice, side);
      if (e2 != cudaSuccess) return e2;
    }
    return cudaSuccess;
  };

  // U12 lookahead (as in the single-GPU schedule, EBV_U12_LA): step K
  // updates block row K+1 of every rank's columns before the rows below, and
  // the side stream solves U12 of step K+1 (after panel K+1's broadcast)
  // while the caller stream updates the rest; per entry the same operations
  // in the same order (bitwise).
  static const int kDistU12La = [] {
    const char* ev = getenv("EBV_U12_LA");
    return ev ? atoi(ev) : -1;
  }();
  const bool u12la = kDistU12La >= 0 ? kDistU12La != 0 : n >= 16384;
  bool u12_done = false;   // U12 of the current step was solved on the side stream

  e = prepare_panel(0);
  if (e != cudaSuccess) return cuda_fail(e, "dist panel");
  for (int64_t K = 0; K < N; K++) {
    const int64_t c0 = K * nb, w = p0.width(K), M = n - c0;
    const int64_t owner = p0.owner(K);
    // ---- broadcast panel K (side stream, step order on every rank)
    if (real) {
      if (K >= 2) {
        e = cudaStreamWaitEvent(side, d->ev_free[K & 1], 0);
        if (e != cudaSuccess) return cuda_fail(e, "dist wait");
      }
      ncclResult_t r = nccl().Broadcast(pbuf(K), pbuf(K), (size_t)(M * w), ncclFloat64, (int)owner, d->comm, side);
      if (r != ncclSuccess) return nccl_fail(r, "ncclBroadcast(panel)");
      c->launches += 1;
    }
    if (u12_done) {   // U12 of this step for every local column after block K, on the side stream
      e = cudaStreamWaitEvent(side, d->ev_brow, 0);
      for (auto& v : views) {
        if (e != cudaSuccess) break;
        const int64_t lc0 = suffix_after(v.plan, K);
        const int64_t ncols = v.plan.cols - lc0;
        if (ncols > 0) e = trsm_l(c, w, ncols, pbuf(K), M, v.A + c0 + lc0 * v.lda, v.lda, side);
      }
      if (e != cudaSuccess) return cuda_fail(e, "dist U12 (lookahead)");
    }
    e = cudaEventRecord(d->ev_ready[K & 1], side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, d->ev_ready[K & 1], 0);
    if (e != cudaSuccess) return cuda_fail(e, "dist order");
    // ---- updates of step K on the caller stream; block K+1 first
    const bool has_next = K + 1 < N;
    const int64_t owner1 = has_next ? p0.owner(K + 1) : -1;
    const int64_t w1 = has_next ? p0.width(K + 1) : 0;
    // the next step takes the lookahead if its block row has rows below it
    const bool la_next = u12la && has_next && M - w > w1;
    for (auto& v : views) {
      const int64_t lc0 = suffix_after(v.plan, K);
      int64_t ncols = v.plan.cols - lc0;
      if (ncols <= 0) continue;
      double* X = v.A + c0 + lc0 * v.lda;
      int64_t first = 0;
      if (has_next && v.plan.rank == owner1) {
        // block K+1 is the first local block after K
        if (!u12_done) e = trsm_l(c, w, w1, pbuf(K), M, X, v.lda, s);
        if (e == cudaSuccess) e = gemm(c, M - w, w1, w, pbuf(K) + w, M, X, v.lda, X + w, v.lda, false, s, KC_UPDATE);
        if (e == cudaSuccess) e = cudaEventRecord(d->ev_next, s);
        if (e != cudaSuccess) return cuda_fail(e, "dist update(next)");
        first = w1;
      }
      if (ncols - first > 0) {
        double* X2 = X + first * v.lda;
        if (!u12_done) e = trsm_l(c, w, ncols - first, pbuf(K), M, X2, v.lda, s);
        if (e == cudaSuccess) {
          const int64_t rows = la_next ? w1 : M - w;   // block row K+1 only, the rest below
          e = gemm(c, rows, ncols - first, w, pbuf(K) + w, M, X2, v.lda, X2 + w, v.lda, false, s, KC_UPDATE);
        }
        if (e != cudaSuccess) return cuda_fail(e, "dist update");
      }
    }
    if (la_next) {
      e = cudaEventRecord(d->ev_brow, s);
      for (auto& v : views) {
        if (e != cudaSuccess) break;
        const int64_t lc0 = suffix_after(v.plan, K);
        int64_t ncols = v.plan.cols - lc0;
        if (ncols <= 0) continue;
        double* X = v.A + c0 + lc0 * v.lda;
        const int64_t first = (v.plan.rank == owner1) ? w1 : 0;
        if (ncols - first <= 0) continue;
        double* X2 = X + first * v.lda;
        e = gemm(c, M - w - w1, ncols - first, w, pbuf(K) + w + w1, M, X2, v.lda, X2 + w + w1, v.lda, false, s,
                 KC_UPDATE);
      }
      if (e != cudaSuccess) return cuda_fail(e, "dist update (rows below)");
    }
    u12_done = la_next;
    e = cudaEventRecord(d->ev_free[K & 1], s);
    if (e != cudaSuccess) return cuda_fail(e, "dist order");
    // ---- lookahead: panel K+1 on the side stream once its columns are updated
    if (has_next) {
      bool mine = false;
      for (auto& v : views) mine = mine || v.plan.rank == owner1;
      if (mine) {
        e = cudaStreamWaitEvent(side, d->ev_next, 0);
        if (e == cudaSuccess) e = prepare_panel(K + 1);
        if (e != cudaSuccess) return cuda_fail(e, "dist panel");
      }
    }
  }
  // join the side stream back into the caller's
  e = cudaEventRecord(d->ev_side, side);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, d->ev_side, 0);
  if (e != cudaSuccess) return cuda_fail(e, "dist join");
  if (real) {
    // first failing step over all owners: min over nonzero info words
    info_to_min_kernel<<<1, 1, 0, s>>>(info);
    ncclResult_t r = nccl().AllReduce(info, info, 1, ncclInt64, ncclMin, d->comm, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(info)");
    info_from_min_kernel<<<1, 1, 0, s>>>(info);
    c->launches += 3;
  }
  return EBV_SUCCESS;
}

// The ring solve.  Forward, K ascending: owner(K) receives the right-hand
// side from owner(K-1), runs one window launch of the wavefront solve kernel
// over its block column K (the diagonal block substituted, the rows below
// updated by the block's columns, per entry in canonical order) and sends the
// right-hand side on to owner(K+1).  Backward mirrors it with K descending.
// Every entry sees the oracle's operation sequence (the ring visits the
// column blocks in order), so X is bitwise the one-GPU result for every P.
ebv_status_t dist_solve(ebv_context* c, ebv_dist_state* d, std::vector<View>& views, int64_t n, double* B,
                        int64_t ldb, int64_t nrhs, cudaStream_t s) {
  const Plan& p0 = views[0].plan;
  const int64_t nb = p0.nb, N = p0.N;
  const bool real = d->comm && (d->nranks > 1 || force_nccl());
  const size_t cnt = (size_t)(ldb * (nrhs - 1) + n);
  if (n <= 0 || nrhs <= 0) return EBV_SUCCESS;
  if (d->nranks == 1 && views.size() == 1 && !(d->comm && force_nccl())) {
    // one rank: its slab is the whole matrix (blocks in ascending order),
    // so the ring has no hop — the single-GPU solve, same per-entry order
    return solve_full(c, n, views[0].A, views[0].lda, B, ldb, nrhs, s);
  }
  auto find = [&](int64_t J) -> View* {
    for (auto& v : views)
      if (v.plan.rank == p0.owner(J)) return &v;
    return nullptr;
  };
  const int64_t G = solve_max_interleave();
  const int64_t groups = (nrhs + G - 1) / G;
  const int64_t NBr = (n + solve_block_rows() - 1) / solve_block_rows();
  const int64_t nflags = 2 * NBr * G * groups, ntick = 2 * N * groups;
  if (nflags + ntick > d->sws_cap) {
    if (d->sws) cudaFree(d->sws);
    d->sws = nullptr;
    d->sws_cap = 0;
    cudaError_t e = cudaMalloc(&d->sws, (nflags + ntick) * sizeof(int));
    if (e != cudaSuccess) { set_error("ring-solve workspace alloc failed"); return EBV_ERR_ALLOC; }
    e = cudaMemset(d->sws, 0, (nflags + ntick) * sizeof(int));
    if (e != cudaSuccess) return cuda_fail(e, "ring-solve workspace");
    d->sws_cap = nflags + ntick;
  }
  int* flags = d->sws;
  int* tick = d->sws + nflags;
  cudaError_t e = cudaMemsetAsync(tick, 0, ntick * sizeof(int), s);
  if (e != cudaSuccess) return cuda_fail(e, "ring-solve tickets");
  // one epoch for the whole ring solve (its flags are per (group, sweep))
  const int ep = (int)(c->solve_epoch % 0x3FFFFFF0) + 1;
  c->solve_epoch++;
  ncclResult_t r = ncclSuccess;
  for (int pass = 0; pass < 2; pass++) {
    const bool fwd = pass == 0;
    for (int64_t t = 0; t < N; t++) {
      const int64_t K = fwd ? t : N - 1 - t;
      View* v = find(K);
      if (!v) continue;
      const int64_t c0 = K * nb, w = p0.width(K);
      const int64_t prev = fwd ? K - 1 : K + 1, next = fwd ? K + 1 : K - 1;
      if (real && prev >= 0 && prev < N && p0.owner(prev) != v->plan.rank) {
        r = nccl().Recv(B, cnt, ncclFloat64, (int)p0.owner(prev), d->comm, s);
        if (r != ncclSuccess) return nccl_fail(r, fwd ? "ncclRecv(fwd)" : "ncclRecv(bwd)");
      }
      const double* Lk = v->A + v->plan.loc[K] * v->lda;
      for (int64_t g = 0; g < groups; g++) {
        const int64_t r0 = g * G, nr = nrhs - r0 < G ? nrhs - r0 : G;
        int* fl = flags + (g * 2 + pass) * NBr * G;
        int* tk = tick + (g * 2 + pass) * N + K;
        e = timed(c, KC_SOLVE, 2.0 * w * (fwd ? n - c0 : c0 + w) * nr, 8.0 * w * (fwd ? n - c0 : c0 + w), s, 1,
                  [&] { return launch_solve_window(n, Lk, v->lda, c0, w, fwd, B + r0 * ldb, ldb, nr, tk, fl, ep, s); });
        if (e != cudaSuccess) return cuda_fail(e, fwd ? "dist forward" : "dist backward");
      }
      if (real && next >= 0 && next < N && p0.owner(next) != v->plan.rank) {
        r = nccl().Send(B, cnt, ncclFloat64, (int)p0.owner(next), d->comm, s);
        if (r != ncclSuccess) return nccl_fail(r, fwd ? "ncclSend(fwd)" : "ncclSend(bwd)");
      }
    }
  }
  if (real) {
    r = nccl().Broadcast(B, B, cnt, ncclFloat64, (int)p0.owner(0), d->comm, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclBroadcast(x)");
  }
  return EBV_SUCCESS;
}

ebv_status_t check_common(ebv_context* c, int64_t n, int64_t lda, int P) {
  if (!c) return invalid("dist: NULL ctx");
  if (n < 0 || P < 1) return invalid("dist: bad size");
  if (lda < (n > 1 ? n : 1)) return invalid("dist: lda < n");
  return EBV_SUCCESS;
}

// The pivot floor of a distributed factorization (before any update): tau
// as given, or (tau < 0) the default n * eps * ||A||_inf (reading R9) from
// the global row absolute sums — each rank sums its local columns (j
// ascending), the partial sums are added over the ranks (ncclAllReduce sum;
// emulation: rank order), and the maximum row sum gives the floor.  For
// inputs whose row sums are exact (the generator's 2^-30 grid) this is
// bitwise the single-GPU floor; otherwise it can differ in the last bits
// (reading R18: the norm's summation order is unspecified).
ebv_status_t dist_tau(ebv_context* c, ebv_dist_state* d, std::vector<View>& views, int64_t n, double tau,
                      cudaStream_t s) {
  cudaError_t e = launch_tau(n, nullptr, n > 0 ? n : 1, tau >= 0 ? tau : 0.0, c->d_tau, c->d_norm, s);
  c->launches += 1;
  if (e != cudaSuccess) return cuda_fail(e, "dist tau");
  if (tau >= 0 || n == 0) return EBV_SUCCESS;
  if (n > c->vec_cap) {
    if (c->d_vec) cudaFree(c->d_vec);
    c->d_vec = nullptr;
    c->vec_cap = 0;
    if (cudaMalloc(&c->d_vec, n * sizeof(double)) != cudaSuccess) { set_error("workspace alloc failed"); return EBV_ERR_ALLOC; }
    c->vec_cap = n;
  }
  bool first = true;
  for (auto& v : views) {
    e = launch_rowabs(n, v.A, v.lda, v.plan.cols, c->d_vec, first, s);
    if (e != cudaSuccess) return cuda_fail(e, "dist row sums");
    c->launches += 1;
    first = false;
  }
  if (d->comm && (d->nranks > 1 || force_nccl())) {
    ncclResult_t r = nccl().AllReduce(c->d_vec, c->d_vec, (size_t)n, ncclFloat64, ncclSum, d->comm, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce(row sums)");
    c->launches += 1;
  }
  e = launch_tau_from_rows(n, c->d_vec, c->d_tau, s);
  c->launches += 1;
  if (e != cudaSuccess) return cuda_fail(e, "dist tau");
  return EBV_SUCCESS;
}

}  // namespace

namespace ebv {
namespace sched {
void dist_release(ebv_context* c) {   // called by ebv_destroy
  if (!c || !c->dist) return;
  if (c->dist->comm && nccl().ok) nccl().CommDestroy(c->dist->comm);
  if (c->dist->pbuf) cudaFree(c->dist->pbuf);
  if (c->dist->sws) cudaFree(c->dist->sws);
  release_events(c->dist);
  delete c->dist;
  c->dist = nullptr;
}
}  // namespace sched
}  // namespace ebv

extern "C" {

ebv_status_t ebv_get_unique_id(void* uid) {
  if (!uid) return invalid("ebv_get_unique_id: NULL");
  if (!nccl().ok) { set_error("libnccl.so.2 could not be loaded"); return EBV_ERR_NCCL; }
  ncclUniqueId id;
  ncclResult_t r = nccl().GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(uid, &id, sizeof(id));
  return EBV_SUCCESS;
}

ebv_status_t ebv_create_dist(ebv_context_t* ctx, int device, const void* uid, int rank, int nranks, int64_t nb,
                             ebv_layout_t layout) {
  if (!ctx || !uid || nranks < 1 || rank < 0 || rank >= nranks) return invalid("ebv_create_dist: bad arguments");
  if (nb <= 0 || nb % 64) return invalid("ebv_create_dist: nb must be a positive multiple of 64");
  if (layout != EBV_LAYOUT_CYCLIC && layout != EBV_LAYOUT_EBVPAIR && layout != EBV_LAYOUT_SNAKE)
    return invalid("ebv_create_dist: bad layout");
  if (!nccl().ok) { set_error("libnccl.so.2 could not be loaded"); return EBV_ERR_NCCL; }
  ebv_status_t st = ebv_create(ctx, device);
  if (st != EBV_SUCCESS) return st;
  DeviceGuard g(device);
  ebv_dist_state* d = new ebv_dist_state();
  d->rank = rank; d->nranks = nranks; d->nb = nb; d->layout = layout;
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclResult_t r = nccl().CommInitRank(&d->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete d;
    ebv_destroy(*ctx);
    *ctx = nullptr;
    return nccl_fail(r, "ncclCommInitRank");
  }
  (*ctx)->dist = d;
  (*ctx)->nb = nb;
  return EBV_SUCCESS;
}

int ebv_dist_nranks(ebv_context_t c) {
  if (!c || !c->dist) return -1;
  if (!c->dist->comm || !nccl().CommCount) return c->dist->nranks;
  int count = -1;
  if (nccl().CommCount(c->dist->comm, &count) != ncclSuccess) return -1;
  return count;
}

ebv_status_t ebv_dist_local_blocks(int64_t n, int64_t nb, int rank, int nranks, ebv_layout_t layout, int64_t* blocks,
                                   int64_t cap, int64_t* nblocks, int64_t* local_cols) {
  if (n < 0 || nb <= 0 || nranks < 1 || rank < 0 || rank >= nranks || !nblocks || !local_cols)
    return invalid("ebv_dist_local_blocks: bad arguments");
  Plan p = make_plan(n, nb, rank, nranks, layout);
  *nblocks = (int64_t)p.blocks.size();
  *local_cols = p.cols;
  if (blocks) {
    if (cap < (int64_t)p.blocks.size()) return invalid("ebv_dist_local_blocks: cap too small");
    for (size_t i = 0; i < p.blocks.size(); i++) blocks[i] = p.blocks[i];
  }
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_factor_dist(ebv_context_t c, int64_t n, double* A_local, int64_t lda, double tau, int64_t* d_info,
                                void* stream) {
  if (!c || !c->dist) return invalid("ebv_lu_factor_dist: not a distributed context");
  ebv_dist_state* d = c->dist;
  ebv_status_t st = check_common(c, n, lda, d->nranks);
  if (st != EBV_SUCCESS) return st;
  if (!d_info) return invalid("ebv_lu_factor_dist: d_info NULL");
  std::vector<View> views{View{make_plan(n, d->nb, d->rank, d->nranks, d->layout), A_local, lda}};
  if (views[0].plan.cols > 0 && !A_local) return invalid("ebv_lu_factor_dist: A_local NULL");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  // CUDA-graph replay, as ebv_lu_factor: the second call with the same
  // arguments captures the schedule (kernels, events and the NCCL
  // collectives, which NCCL supports in captured streams; every rank
  // captures and replays the same collective sequence), later calls replay
  // it (EBV_DIST_GRAPHS=0: launch directly every time)
  static const bool kDistGraphs = [] {
    const char* ev = getenv("EBV_DIST_GRAPHS");
    return !(ev && atoi(ev) == 0);
  }();
  ebv_context::GraphEntry* ge = nullptr;
  const bool use_graph = kDistGraphs && c->graphs && !c->stats && s != nullptr && n > 0;
  if (use_graph) {
    for (auto& en : c->gcache)
      if (en.n == n && en.lda == lda && en.A == A_local && en.info == d_info && en.tau == tau && en.nb == d->nb &&
          en.leaf == c->leaf && en.la == c->lookahead) {
        ge = &en;
        break;
      }
    if (ge && ge->exec) {
      cudaError_t e = cudaGraphLaunch(ge->exec, s);
      if (e != cudaSuccess) return cuda_fail(e, "dist graph launch");
      c->launches += ge->launches;
      return EBV_SUCCESS;
    }
    if (!ge) {
      if (c->gcache.size() >= 8) {
        if (c->gcache.front().exec) cudaGraphExecDestroy(c->gcache.front().exec);
        c->gcache.erase(c->gcache.begin());
      }
      c->gcache.push_back({n, lda, d->nb, c->leaf, A_local, d_info, tau, c->lookahead, 0, 0, nullptr});
      ge = &c->gcache.back();
    }
    ge->hits++;
  }
  auto run = [&]() -> ebv_status_t {
    cudaError_t e = launch_set_info0(d_info, s);
    if (e != cudaSuccess) return cuda_fail(e, "dist init");
    c->launches += 1;
    ebv_status_t r = dist_tau(c, d, views, n, tau, s);
    if (r == EBV_SUCCESS && n > 0) r = dist_factor(c, d, views, n, d_info, s);
    return r;
  };
  const bool capture = use_graph && ge && ge->hits >= 2;
  if (!capture) return run();
  const int64_t l0 = c->launches;
  bool ok = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  st = ok ? run() : EBV_ERR_CUDA;
  cudaGraph_t graph = nullptr;
  if (ok) ok = cudaStreamEndCapture(s, &graph) == cudaSuccess && st == EBV_SUCCESS;
  if (ok) ok = cudaGraphInstantiateWithFlags(&ge->exec, graph, cudaGraphInstantiateFlagUseNodePriority) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  if (!ok) {
    // the capture failed (nothing of it ran): never capture these arguments
    // again and run the schedule directly
    (void)cudaGetLastError();
    ge->exec = nullptr;
    ge->hits = INT32_MIN / 2;
    return run();
  }
  ge->launches = c->launches - l0;
  cudaError_t ec = cudaGraphLaunch(ge->exec, s);
  if (ec != cudaSuccess) return cuda_fail(ec, "dist graph launch");
  return EBV_SUCCESS;
}

ebv_status_t ebv_lu_solve_dist(ebv_context_t c, int64_t n, const double* LU_local, int64_t lda, double* B, int64_t ldb,
                               int64_t nrhs, void* stream) {
  if (!c || !c->dist) return invalid("ebv_lu_solve_dist: not a distributed context");
  ebv_dist_state* d = c->dist;
  ebv_status_t st = check_common(c, n, lda, d->nranks);
  if (st != EBV_SUCCESS) return st;
  if (nrhs < 0 || ldb < (n > 1 ? n : 1)) return invalid("ebv_lu_solve_dist: bad B");
  if (n == 0 || nrhs == 0) return EBV_SUCCESS;
  if (!B) return invalid("ebv_lu_solve_dist: B NULL");
  DeviceGuard g(c->device);
  std::vector<View> views{View{make_plan(n, d->nb, d->rank, d->nranks, d->layout), const_cast<double*>(LU_local), lda}};
  return dist_solve(c, d, views, n, B, ldb, nrhs, (cudaStream_t)stream);
}

ebv_status_t ebv_lu_factor_dist_emulated(ebv_context_t c, int64_t n, int nranks, int64_t nb, ebv_layout_t layout,
                                         double* const* slabs, int64_t lda, double tau, int64_t* d_info, void* stream) {
  ebv_status_t st = check_common(c, n, lda, nranks);
  if (st != EBV_SUCCESS) return st;
  if (nb <= 0 || nb % 64) return invalid("emulated: nb must be a positive multiple of 64");
  if (!d_info || (n > 0 && !slabs)) return invalid("emulated: NULL pointer");
  DeviceGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_set_info0(d_info, s);
  if (e != cudaSuccess) return cuda_fail(e, "emulated init");
  ebv_dist_state tmp;
  tmp.nranks = nranks; tmp.nb = nb; tmp.layout = layout;
  std::vector<View> views;
  for (int r = 0; r < nranks; r++) views.push_back(View{make_plan(n, nb, r, nranks, layout), slabs[r], lda});
  st = dist_tau(c, &tmp, views, n, tau, s);
  if (st != EBV_SUCCESS || n == 0) return st;
  st = dist_factor(c, &tmp, views, n, d_info, s);
  cudaStreamSynchronize(s);   // the temporary panel buffers / events die with tmp
  if (tmp.pbuf) cudaFree(tmp.pbuf);
  release_events(&tmp);
  return st;
}

ebv_status_t ebv_lu_solve_dist_emulated(ebv_context_t c, int64_t n, int nranks, int64_t nb, ebv_layout_t layout,
                                        double* const* slabs, int64_t lda, double* B, int64_t ldb, int64_t nrhs,
                                        void* stream) {
  ebv_status_t st = check_common(c, n, lda, nranks);
  if (st != EBV_SUCCESS) return st;
  if (nb <= 0 || nb % 64) return invalid("emulated: nb must be a positive multiple of 64");
  if (nrhs < 0 || ldb < (n > 1 ? n : 1)) return invalid("emulated: bad B");
  if (n == 0 || nrhs == 0) return EBV_SUCCESS;
  if (!B || !slabs) return invalid("emulated: NULL pointer");
  DeviceGuard g(c->device);
  ebv_dist_state tmp;
  tmp.nranks = nranks; tmp.nb = nb; tmp.layout = layout;
  std::vector<View> views;
  for (int r = 0; r < nranks; r++) views.push_back(View{make_plan(n, nb, r, nranks, layout), slabs[r], lda});
  st = dist_solve(c, &tmp, views, n, B, ldb, nrhs, (cudaStream_t)stream);
  // the temporary solve workspace dies with tmp (after the launches using it)
  cudaStreamSynchronize((cudaStream_t)stream);
  if (tmp.sws) cudaFree(tmp.sws);
  return st;
}

}  // extern "C"
