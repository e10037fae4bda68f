// k_vector.cu — the paper's vector-level elimination (EBV_PATH_VECTOR):
// Eq 6-a..c executed step by step, with the EbV equal-length
// pairing (Eq 7) as the column -> CTA owner map.
//
// One persistent cooperative kernel.  Columns are grouped in blocks of bw
// consecutive columns; block pairs {J, Nb-1-J} (first with last: the paired
// blocks' on-or-below-diagonal lengths sum to a constant, reading R12) are
// dealt round-robin to the CTAs, which keep their columns resident in shared
// memory for the whole factorization.  Block J's steps k:
//   * the owner of block J runs them locally: Eq 6-a on column k (the L_(k)
//     vector), Eq 6-c on the block's later columns with the U_(k) row
//     entries it holds, writes the block's columns to A and publishes one
//     release flag per block;
//   * every other CTA acquires the flag, reads the block's L_(k) vectors from
//     L2 and applies the bw rank-1 updates, in ascending k, to its columns
//     of later blocks.
// Lookahead: the owner of block J+1 applies block J to that block first,
// then factors and publishes it, and only then updates its remaining
// columns — so the dependent chain per block is one flag hop plus bw local
// steps.  Inside a block the owner factors the bw x bw diagonal block in one
// warp (shuffles carry the pivot row), then every row below runs the bw
// steps in its own thread, dividing by a hoisted reciprocal with a verified
// Markstein correction (true division when unverified).  Per entry the
// arithmetic is the oracle's (bitwise); `cyclic` selects the plain J mod C
// block map for comparison.  Measured per-block chain (probes/vector_trace,
// n = 1024): flag hop ~0.5 us, apply ~3.5 us, diagonal block ~3 us (eight
// dependent divisions), rows below ~3.5 us.
#include "ebv_internal.cuh"
#include "ebv_device.cuh"

#include <cstdlib>
#include <type_traits>

namespace ebv {
namespace {

constexpr int VT = 512;   // threads per CTA

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
// acquire polls: the invalidation of L1 an acquire load implies costs
// nothing here (the CTA reads other CTAs' data only through L2), and it
// saves the extra round trip of a relaxed poll followed by a fence
__device__ __forceinline__ void wait_flag(const int* p, int v) {
  int t;
  dev::SpinGuard g;
  do {
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(t) : "l"(p) : "memory");
    g.poll();
  } while (t != v);
}

// q = RN(y/u) from r = RN(1/u) by one Markstein correction; `ok` is cleared
// unless the exact remainder proves q correctly rounded (then the caller
// redoes the row with true division) — same test as k_solve.cu's quot().
__device__ __forceinline__ double quot(double y, double u, double r, bool& ok) {
  const double q = dev::quot_mk(y, u, r);
  ok = ok && dev::quot_is_rn(y, u, q);
  return q;
}

// owner CTA of column block J: blocks are grouped in chunks of cb
// consecutive blocks (a chunk's blocks hand over to each other inside one
// CTA, from shared memory); chunk pairs {i, Nc-1-i} (first with last) are
// dealt round-robin, or chunk i -> i mod C (cyclic)
__device__ __forceinline__ int block_owner(int J, int Nb, int C, int cyclic, int cb) {
  const int ch = J / cb, Nc = (Nb + cb - 1) / cb;
  if (cyclic) return ch % C;
  const int p = ch < Nc - 1 - ch ? ch : Nc - 1 - ch;
  return p % C;
}

#ifdef EBV_VECTOR_TRACE
// probes/vector_trace.cu: per-block phase timestamps (%globaltimer, ns)
__device__ unsigned long long g_vtrace[2048][6];
#define EBV_VTR(J, slot)                                                            \
  do {                                                                             \
    __syncthreads();                                                               \
    if (tid == 0 && (J) < 2048) {                                                  \
      unsigned long long t;                                                        \
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));                        \
      g_vtrace[J][slot] = t;                                                       \
    }                                                                              \
  } while (0)
#else
#define EBV_VTR(J, slot) \
  do {                   \
  } while (0)
#endif

constexpr int BWMAX = 8;   // block width limit

// The kernel body runs once per block with little work per thread, so it is
// instruction-fetch sensitive: loops over rows and columns stay rolled and
// only the bw-long step loops are unrolled (a fully unrolled variant was 10k
// SASS instructions and 8x slower per block).
__global__ void __launch_bounds__(VT, 1)
    vector_lu_kernel(int n, double* __restrict__ A, int64_t lda, const double* __restrict__ tau,
                     unsigned long long* info_min, int* flags, int epoch, int cyclic, int bw, int maxcols,
                     int cb) {
  extern __shared__ double scol[];         // owned columns [maxcols][n]
  __shared__ int cols[1024];               // owned global column indices (ascending)
  __shared__ double srcp[BWMAX];           // RN(1/u_kk) of the block being factored
  __shared__ int ncols_s;
  const int C = gridDim.x, me = blockIdx.x, tid = threadIdx.x;
  const int Nb = (n + bw - 1) / bw;
  if (tid == 0) {
    int c = 0;
    for (int J = 0; J < Nb; J++)
      if (block_owner(J, Nb, C, cyclic, cb) == me)
        for (int j = J * bw; j < n && j < (J + 1) * bw; j++) cols[c++] = j;
    ncols_s = c;
  }
  __syncthreads();
  const int ncols = ncols_s;
  {   // owned columns into shared memory, eight loads in flight per thread
      // (a load -> store loop waits one memory round trip per iteration)
    const int total = ncols * n;
    for (int e0 = tid; e0 < total; e0 += 8 * VT) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int e = e0 + u * VT;
        v[u] = e < total ? A[e % n + (int64_t)cols[e / n] * lda] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const int e = e0 + u * VT;
        if (e < total) scol[e] = v[u];
      }
    }
  }
  __syncthreads();
  const double tv = *tau;

  // slot of the first owned column >= j (columns are ascending)
  auto first_slot = [&](int j) -> int {
    int lo = 0, hi = ncols;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (cols[mid] < j) lo = mid + 1; else hi = mid;
    }
    return lo;
  };

  // Apply the steps k0..k1-1 (block J's L_(k) vectors at lsrc + (k-k0)*n) to
  // owned columns in slots [c0, c1) (Eq 6-c).  Every entry still receives
  // its fma's in ascending k: phase A finishes rows k0+1..k1-1 of each
  // column (the U_(k) row entries the later steps multiply by), phase B then
  // runs each row i >= k1 through all of the block's steps.
  auto apply = [&](int k0, int k1, const double* lsrc, int64_t lstr, int c0, int c1) {
    if (c0 >= c1) return;
    const int nbk = k1 - k0;
#pragma unroll 1
    for (int c = c0 + tid; c < c1; c += VT) {      // phase A: one thread per column
      double* col = scol + (size_t)c * n + k0;
      double a[BWMAX];
#pragma unroll
      for (int ii = 0; ii < BWMAX; ii++) a[ii] = ii < nbk ? col[ii] : 0.0;
#pragma unroll
      for (int kk = 0; kk < BWMAX - 1; kk++)
#pragma unroll
        for (int ii = kk + 1; ii < BWMAX; ii++)
          if (ii < nbk) a[ii] = fma(-lsrc[kk * lstr + k0 + ii], a[kk], a[ii]);
#pragma unroll
      for (int ii = 1; ii < BWMAX; ii++)
        if (ii < nbk) col[ii] = a[ii];
    }
    __syncthreads();
#pragma unroll 1
    for (int i = k1 + tid; i < n; i += VT) {       // phase B: rows >= k1
      double l[BWMAX];
#pragma unroll
      for (int kk = 0; kk < BWMAX; kk++) l[kk] = kk < nbk ? lsrc[kk * lstr + i] : 0.0;
      int c = c0;
#pragma unroll 1
      for (; c + 3 < c1; c += 4) {                 // four independent chains per thread
        double* p0 = scol + (size_t)c * n;
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; q++) v[q] = p0[(size_t)q * n + i];
#pragma unroll
        for (int kk = 0; kk < BWMAX; kk++)
          if (kk < nbk)
#pragma unroll
            for (int q = 0; q < 4; q++) v[q] = fma(-l[kk], p0[(size_t)q * n + k0 + kk], v[q]);
#pragma unroll
        for (int q = 0; q < 4; q++) p0[(size_t)q * n + i] = v[q];
      }
#pragma unroll 1
      for (; c < c1; c++) {
        double* p0 = scol + (size_t)c * n;
        double v0 = p0[i];
#pragma unroll
        for (int kk = 0; kk < BWMAX; kk++)
          if (kk < nbk) v0 = fma(-l[kk], p0[k0 + kk], v0);
        p0[i] = v0;
      }
    }
    __syncthreads();
  };

  // Factor owned block J (its columns are up to date through step J*bw-1),
  // write its rows >= J*bw to A and publish flag[J].  Phase A: the bw x bw
  // diagonal block by the first bw lanes of warp 0 (row k0+r per lane, Eq
  // 6-a/6-c with the pivot row broadcast by shuffles, Eq 6-b); phase B:
  // every row i >= k1 through the block's steps in its own thread — per
  // entry the same fma chain then division as the step-by-step order.
  auto factor_block = [&](int J) {
    const int k0 = J * bw, k1 = min(n, (J + 1) * bw), nbk = k1 - k0;
    const int s0 = first_slot(k0);
    EBV_VTR(J, 1);
    double* blk = scol + (size_t)s0 * n;           // column c of the block at blk + c*n
    if (tid < 32) {
      const int r = tid;
      double a[BWMAX];
#pragma unroll
      for (int c = 0; c < BWMAX; c++) a[c] = (r < nbk && c < nbk) ? blk[(size_t)c * n + k0 + r] : 0.0;
#pragma unroll
      for (int kk = 0; kk < BWMAX; kk++) {
        if (kk < nbk) {
          const double piv = __shfl_sync(0xffffffffu, a[kk], kk);
          if (r == 0 && fabs(piv) <= tv) atomicMin(info_min, (unsigned long long)(k0 + kk + 1));
          const bool below = r > kk && r < nbk;
          if (below) a[kk] = a[kk] / piv;                               // Eq 6-a
#pragma unroll
          for (int c = kk + 1; c < BWMAX; c++) {
            const double u = __shfl_sync(0xffffffffu, a[c], kk);        // Eq 6-b
            if (below && c < nbk) a[c] = fma(-a[kk], u, a[c]);          // Eq 6-c
          }
        }
      }
      if (r < nbk) {
#pragma unroll
        for (int c = 0; c < BWMAX; c++)
          if (c < nbk) {
            blk[(size_t)c * n + k0 + r] = a[c];
            A[k0 + r + (int64_t)(k0 + c) * lda] = a[c];
          }
        double d = a[0];
#pragma unroll
        for (int c = 1; c < BWMAX; c++)
          if (c == r) d = a[c];
        srcp[r] = 1.0 / d;
      }
    }
    __syncthreads();
    EBV_VTR(J, 2);
    // rows below: the quotient from the hoisted reciprocal, verified; rows
    // with an unverified step are redone with true division
    // (two rows per thread at a time, for overlap of their dependent chains)
    auto below_rows = [&](int i0, auto exact_tag) {
      constexpr bool exact = decltype(exact_tag)::value;
      double a[2][BWMAX];
      bool ok[2] = {true, true};
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int i = i0 + h * VT;
#pragma unroll
        for (int c = 0; c < BWMAX; c++) a[h][c] = (c < nbk && i < n) ? blk[(size_t)c * n + i] : 0.0;
      }
#pragma unroll
      for (int kk = 0; kk < BWMAX; kk++) {
        if (kk < nbk) {
          const double u = blk[(size_t)kk * n + k0 + kk], rp = srcp[kk];
#pragma unroll
          for (int h = 0; h < 2; h++) a[h][kk] = exact ? a[h][kk] / u : quot(a[h][kk], u, rp, ok[h]);   // Eq 6-a
#pragma unroll
          for (int c = kk + 1; c < BWMAX; c++)
            if (c < nbk) {
              const double uc = blk[(size_t)c * n + k0 + kk];
#pragma unroll
              for (int h = 0; h < 2; h++) a[h][c] = fma(-a[h][kk], uc, a[h][c]);                    // Eq 6-c
            }
        }
      }
      const bool good = ok[0] && (ok[1] || i0 + VT >= n);
      if (good) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int i = i0 + h * VT;
          if (i < n)
#pragma unroll
            for (int c = 0; c < BWMAX; c++)
              if (c < nbk) {
                blk[(size_t)c * n + i] = a[h][c];
                A[i + (int64_t)(k0 + c) * lda] = a[h][c];
              }
        }
      }
      return good;
    };
#pragma unroll 1
    for (int i = k1 + tid; i < n; i += 2 * VT)
      if (!below_rows(i, std::false_type{})) below_rows(i, std::true_type{});
    __syncthreads();
    EBV_VTR(J, 3);
    if (tid == 0) st_release(flags + J, epoch);
    EBV_VTR(J, 4);
  };

  if (block_owner(0, Nb, C, cyclic, cb) == me) factor_block(0);
  for (int J = 0; J < Nb - 1; J++) {
    const int k0 = J * bw, k1 = min(n, (J + 1) * bw);
    const int c1 = first_slot(k1);                  // first owned column after block J
    if (c1 >= ncols) break;                         // nothing of mine is updated by block J or later
    const double* lsrc;
    int64_t lstr = n;
    if (block_owner(J, Nb, C, cyclic, cb) == me) {
      lsrc = scol + (size_t)first_slot(k0) * n;    // block J's columns, final here
    } else {
      if (tid == 0) wait_flag(flags + J, epoch);
      __syncthreads();
      // read its L_(k) vectors in place from L2: the acquire above ordered
      // them, and the acquire's L1 invalidation leaves no stale line (staging
      // them in shared memory first cost a further ~4 us per block)
      lsrc = A + (int64_t)k0 * lda;
      lstr = lda;
    }
    if (block_owner(J + 1, Nb, C, cyclic, cb) == me) {
      EBV_VTR(J + 1, 0);
      // lookahead: block J+1 first, factor + publish it, then the rest
      const int c2 = first_slot(min(n, (J + 2) * bw));
      apply(k0, k1, lsrc, lstr, c1, c2);
      factor_block(J + 1);
      apply(k0, k1, lsrc, lstr, c2, ncols);
    } else {
      apply(k0, k1, lsrc, lstr, c1, ncols);
    }
  }
  // the U part (rows above each owned block) was completed in shared memory
  for (int c = 0; c < ncols; c++) {
    const int j = cols[c], top = (j / bw) * bw;
    for (int i = tid; i < top; i += VT) A[i + (int64_t)j * lda] = scol[(size_t)c * n + i];
  }
}

__global__ void info_finalize_kernel(const unsigned long long* info_min, int64_t* info) {
  unsigned long long v = *info_min;
  *info = (v == ~0ull) ? 0 : (int64_t)v;
}

int chunk_blocks() {   // EBV_VECTOR_CHUNK: consecutive blocks per owner chunk (default 1)
  static int v = [] {
    const char* e = getenv("EBV_VECTOR_CHUNK");
    const int c = e ? atoi(e) : 1;
    return c > 0 ? c : 1;
  }();
  return v;
}

int max_cols(int64_t n, int C, int cyclic, int bw) {
  const int64_t cb = chunk_blocks();
  const int64_t Nb = (n + bw - 1) / bw, Nc = (Nb + cb - 1) / cb;
  if (cyclic) return (int)(((Nc + C - 1) / C) * cb * bw);
  const int64_t pairs = (Nc + 1) / 2;
  return (int)(2 * ((pairs + C - 1) / C) * cb * bw);
}

int clamp_ctas(int64_t n, int num_ctas, int bw) {
  const int cyclic = num_ctas < 0 ? 1 : 0;
  int C = num_ctas < 0 ? -num_ctas : num_ctas;
  const int64_t cb = chunk_blocks();
  const int64_t Nb = (n + bw - 1) / bw, Nc = (Nb + cb - 1) / cb;
  const int64_t units = cyclic ? Nc : (Nc + 1) / 2;
  if (C > units) C = (int)units;
  if (C < 1) C = 1;
  return C;
}

size_t smem_for(int64_t n, int num_ctas, int bw) {
  const int cyclic = num_ctas < 0 ? 1 : 0;
  const int C = clamp_ctas(n, num_ctas, bw);
  return (size_t)max_cols(n, C, cyclic, bw) * n * 8;
}

// largest block width in {8, 4, 2, 1} whose shared-memory image fits
int pick_bw(int64_t n, int num_ctas) {
  int smem_max = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  for (int bw = 8; bw >= 1; bw >>= 1)
    if (max_cols(n, clamp_ctas(n, num_ctas, bw), num_ctas < 0, bw) <= 1024 &&
        smem_for(n, num_ctas, bw) + 9000 <= (size_t)smem_max)
      return bw;
  return 0;
}

}  // namespace

size_t vector_smem_bytes(int64_t n, int num_ctas) {
  const int bw = pick_bw(n, num_ctas);
  return bw ? smem_for(n, num_ctas, bw) : (size_t)1 << 40;
}

int vector_max_ctas(int device, int64_t n) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  (void)n;
  return sms;   // clamped to the number of block pairs at launch
}

cudaError_t launch_vector_lu(int64_t n, double* A, int64_t lda, const double* tau, int64_t* info, int* flags_ws,
                             double* lbuf_ws, int num_ctas, int epoch, cudaStream_t s) {
  // lbuf_ws is used as the 8-byte info accumulator (min over failing steps)
  unsigned long long* info_min = reinterpret_cast<unsigned long long*>(lbuf_ws);
  cudaError_t e = cudaMemsetAsync(info_min, 0xFF, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  if (n <= 0) {
    info_finalize_kernel<<<1, 1, 0, s>>>(info_min, info);
    return cudaGetLastError();
  }
  const int cyclic = num_ctas < 0 ? 1 : 0;
  const int bw = pick_bw(n, num_ctas);
  if (bw == 0) return cudaErrorInvalidValue;
  const int C = clamp_ctas(n, num_ctas, bw);
  const int mc = max_cols(n, C, cyclic, bw);
  const size_t smem = smem_for(n, num_ctas, bw);
  e = cudaFuncSetAttribute(vector_lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int nn = (int)n, ep = epoch, cy = cyclic, bwv = bw, mcv = mc, cbv = chunk_blocks();
  void* args[] = {&nn, &A, &lda, (void*)&tau, &info_min, &flags_ws, &ep, &cy, &bwv, &mcv, &cbv};
  e = cudaLaunchCooperativeKernel((void*)vector_lu_kernel, dim3(C), dim3(VT), args, smem, s);
  if (e != cudaSuccess) return e;
  info_finalize_kernel<<<1, 1, 0, s>>>(info_min, info);
  return cudaGetLastError();
}

}  // namespace ebv

EBV_DEBUG_SETTER(set_debug_vector)
