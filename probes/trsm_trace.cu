// probes/trsm_trace.cu — %clock64 phases of trsm_ru_kernel (k_leaf.cu
// compiled with EBV_LEAF_TRACE): U staging, reciprocals, X loads, and each
// 8-step block of the row-parallel L21 = A21 U11^-1 solve, for one CTA
// (m = 64) and a full grid (m = 8192).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1907_05767_b200/csrc \
//     probes/trsm_trace.cu -o probes/trsm_trace -Lpaper_1907_05767_b200 -lebv \
//     -Xlinker -rpath,\$ORIGIN/../paper_1907_05767_b200
#define EBV_LEAF_TRACE 1
#include "k_leaf.cu"
#include <cstdio>
#include <vector>
#include <cstdlib>
#include <cmath>
#include <cstdint>
// this executable's own kernels need their attribute set through its own
// runtime (libebv.so carries a separate static cudart)
namespace ebv {
cudaError_t ensure_max_dyn_smem(const void* fn, int bytes) {
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
}  // namespace ebv
int main() {
  const int64_t ld = 8192 + 64;
  std::vector<double> h(ld * 64);
  for (int64_t c = 0; c < 64; c++)
    for (int64_t r = 0; r < ld; r++) h[r + c * ld] = (r == c) ? 65.0 : ((r * 7 + c * 13) % 17 - 8) * 1e-2;
  if (getenv("EBV_PROBE_REAL")) {   // generator-like values: k * 2^-30, diag = row sum + 1
    uint64_t st = 88172645463325252ull;
    for (int64_t c = 0; c < 64; c++)
      for (int64_t r = 0; r < ld; r++) {
        st ^= st << 13; st ^= st >> 7; st ^= st << 17;
        h[r + c * ld] = (double)((int64_t)(st % (1ull << 31)) - (1ll << 30)) * 9.313225746154785e-10;
      }
    for (int64_t r = 0; r < 64; r++) { double sum = 1.0; for (int64_t c = 0; c < 64; c++) if (c != r) sum += fabs(h[r + c * ld]); h[r + r * ld] = sum; }
  }
  double* d;
  cudaMalloc(&d, ld * 64 * 8);
  for (int64_t m : {64, 1024, 8192}) {
    for (int rep = 0; rep < 3; rep++) {
      cudaMemcpy(d, h.data(), ld * 64 * 8, cudaMemcpyHostToDevice);
      ebv::launch_trsm_right_upper(m, 64, d + 64, ld, d, ld, 0);
      cudaDeviceSynchronize();
    }
    long long t[16];
    cudaMemcpyFromSymbol(t, ebv::g_ltrace, sizeof(t));
    printf("m %5lld: stage U %lld, rcp %lld, X load %lld, blocks:", (long long)m, t[1] - t[0], t[2] - t[1], t[3] - t[2]);
    for (int b = 0; b < 8; b++) printf(" %lld", t[4 + b] - (b ? t[3 + b] : t[3]));
    printf("  total %lld cycles\n", t[11] - t[0]);
  }
  // the fused panel leaf (diagonal block in every CTA, then its 64 rows below)
  int* cnt; cudaMalloc(&cnt, 4); cudaMemset(cnt, 0, 4);
  double* tau; cudaMalloc(&tau, 8); cudaMemset(tau, 0, 8);
  int64_t* info; cudaMalloc(&info, 8); cudaMemset(info, 0, 8);
  for (int64_t M : {64, 1024, 4096}) {
    for (int rep = 0; rep < 3; rep++) {
      cudaMemcpy(d, h.data(), ld * 64 * 8, cudaMemcpyHostToDevice);
      cudaError_t e = ebv::launch_panel_leaf(M, 64, d, ld, tau, info, 0, cnt, 0);
      cudaError_t e2 = cudaDeviceSynchronize();
      if (e != cudaSuccess || e2 != cudaSuccess) printf("launch %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
    }
    long long t[16];
    cudaMemcpyFromSymbol(t, ebv::g_ltrace, sizeof(t));
    if (getenv("EBV_PANEL_BLK") && atoi(getenv("EBV_PANEL_BLK")) == 0) {
      printf("panel_leaf M %5lld: load+arrive %lld, diag %lld, rcp %lld, x0 load %lld, rows below %lld, total %lld cycles\n",
             (long long)M, t[1] - t[0], t[2] - t[1], t[3] - t[2], t[4] - t[3], t[5] - t[4], t[5] - t[0]);
    } else {
      printf("panel_blk M %5lld: load %lld;", (long long)M, t[1] - t[0]);
      for (int sp = 0; sp < 4; sp++)
        printf(" [A %lld B %lld C %lld]", t[2 + 3 * sp] - (sp ? t[1 + 3 * sp] : t[1]), t[3 + 3 * sp] - t[2 + 3 * sp],
               t[4 + 3 * sp] - t[3 + 3 * sp]);
      printf(" total %lld cycles\n", t[13] - t[0]);
    }
  }
  {   // schedule-like: a 1024 x 1024 matrix, lda 1024, panels at c0 = 0, 64, ... (events)
    const int64_t n = 1024;
    std::vector<double> hm(n * n);
    for (int64_t c = 0; c < n; c++)
      for (int64_t r = 0; r < n; r++) hm[r + c * n] = (r == c) ? 600.0 : ((r * 7 + c * 13) % 17 - 8) * 1e-2;
    double* dm; cudaMalloc(&dm, n * n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int64_t c0 : {0, 64, 512, 896}) {
      float best = 1e9;
      for (int rep = 0; rep < 5; rep++) {
        cudaMemcpy(dm, hm.data(), n * n * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        ebv::launch_panel_leaf(n - c0, 64, dm + c0 + c0 * n, n, tau, info, c0, cnt, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("schedule-like panel c0 %4lld M %4lld: %.2f us (%s)\n", (long long)c0, (long long)(n - c0), best * 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
