// probes/chain_trace.cu — %globaltimer timeline of the chain-pipelined solve
// (k_solve2.cu compiled with EBV_CHAIN_TRACE): per logical step t, the
// chain CTA's pickup / absorbed tiles / diag-tile wait / solve / loader /
// publisher stamps.  Input: a synthetic unit-lower / DD-upper factor (timing
// only, not a parity check).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//     -I<nccl include> probes/chain_trace.cu -o probes/chain_trace \
//     -Lpaper_1907_05767_b200 -lebv -Xlinker -rpath,\$ORIGIN/../paper_1907_05767_b200
#define EBV_CHAIN_TRACE 1
#include "../paper_1907_05767_b200/csrc/k_solve2.cu"
#include "../paper_1907_05767_b200/csrc/k_util.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8192;
  const int nrhs = argc > 2 ? atoi(argv[2]) : 1;
  const int fwd_only = 0;
  std::vector<double> h(n * n);
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) h[i + j * n] = (i == j) ? 2.0 + (i % 7) : ((i * 31 + j * 17) % 13 - 6) * 1e-4;
  double *LU, *B;
  int* flags;
  cudaMalloc(&LU, n * n * 8);
  cudaMalloc(&B, n * 8 * nrhs);
  cudaMalloc(&flags, 2 * ebv::solve_chain_flags(n) * 4);
  cudaMemset(flags, 0, 2 * ebv::solve_chain_flags(n) * 4);
  cudaMemcpy(LU, h.data(), n * n * 8, cudaMemcpyHostToDevice);
  std::vector<double> b(n * nrhs, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; rep++) {
    cudaMemcpy(B, b.data(), n * 8 * nrhs, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    cudaError_t e = ebv::launch_solve_chain(n, LU, n, B, n, nrhs, flags, 100 * rep, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d: %.3f ms (%s)\n", rep, ms, cudaGetErrorString(e == cudaSuccess ? cudaDeviceSynchronize() : e));
  }
  // the trace holds the last sweep run (backward); rerun forward only if asked
  static unsigned long long ct[4096][14];
  cudaMemcpyFromSymbol(ct, ebv::g_ct, sizeof(ct));
  const int64_t NB = (n + 63) / 64;
  unsigned long long t0 = ~0ull;
  for (int64_t t = 0; t < NB && t < 4096; t++)
    for (int k = 0; k < 14; k++)
      if (ct[t][k] && ct[t][k] < t0) t0 = ct[t][k];
  printf("backward sweep (logical steps); us from first stamp\n");
  printf("   t  pick  got  tile0 tile1 tile2 tile3 tile4  wait  diag  sdone  load  pub  hlast  hpub\n");
  for (int64_t t = 0; t < NB && t < 4096; t++) {
    if (t > 24 && t < NB - 4 && t % 16) continue;
    printf("%4lld", (long long)t);
    for (int k = 0; k < 14; k++) printf(" %6.2f", ct[t][k] ? (ct[t][k] - t0) * 1e-3 : -1.0);
    printf("\n");
  }
  static unsigned long long cq[64][4];
  cudaMemcpyFromSymbol(cq, ebv::g_cq, sizeof(cq));
  printf("block %d quarters (us, relative to q0 start): start  loaded  applied  done | load apply done\n", EBV_CQ_T);
  for (int q = 0; q < 16; q++) {
    auto r = [&](int k) { return (cq[q][k] - cq[0][0]) * 1e-3; };
    printf("q%2d %7.3f %7.3f %7.3f %7.3f | %6.3f %6.3f %6.3f\n", q, r(0), r(1), r(2), r(3), r(1) - r(0), r(2) - r(1), r(3) - r(2));
  }
  (void)fwd_only;
  return 0;
}
