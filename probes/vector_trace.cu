// Probe: timeline of the vector path (per block J, on the CTA owning J:
// flag J-1 seen, apply done, diagonal block done, rows below done, released)
// via %globaltimer.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 probes/vector_trace.cu -o probes/vector_trace \
//     -Lpaper_1907_05767_b200 -lebv -Xlinker -rpath,\$ORIGIN/../paper_1907_05767_b200
#define EBV_VECTOR_TRACE 1
#include "../paper_1907_05767_b200/csrc/k_vector.cu"
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 1024;
  int ctas = argc > 2 ? atoi(argv[2]) : 148;
  std::vector<double> hA((size_t)n * n);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) hA[i + j * n] = (i == j) ? 2.0 * n : u(rng);
  double *dA, *tau, *lbuf;
  int64_t* info;
  int* flags;
  cudaMalloc(&dA, (size_t)n * n * 8);
  cudaMalloc(&tau, 8);
  cudaMalloc(&lbuf, 64);
  cudaMalloc(&info, 8);
  cudaMalloc(&flags, n * 4);
  cudaMemset(tau, 0, 8);
  cudaMemset(flags, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 1; rep <= 3; rep++) {
    cudaMemcpy(dA, hA.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    cudaError_t e = ebv::launch_vector_lu(n, dA, n, tau, info, flags, lbuf, ctas, rep, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d vector %.3f ms (launch %s, after %s)\n", rep, ms, cudaGetErrorString(e),
           cudaGetErrorString(cudaGetLastError()));
  }
  static unsigned long long tr[2048][6];
  cudaMemcpyFromSymbol(tr, ebv::g_vtrace, sizeof(tr));
  const int bw = ebv::pick_bw(n, ctas);
  const int64_t Nb = (n + bw - 1) / bw;
  unsigned long long t0 = tr[0][1];
  printf("bw %d Nb %lld; per block J: seen(J-1) apply_done diag_done below_done released (us from block 0 start)\n", bw,
         (long long)Nb);
  for (int64_t J = 0; J < Nb && J < 2048; J++)
    if (J < 8 || J % 16 == 0 || J > Nb - 4)
      printf("  %5lld: %9.2f %9.2f %9.2f %9.2f %9.2f\n", (long long)J, J ? (tr[J][0] - (double)t0) / 1e3 : 0.0,
             (tr[J][1] - (double)t0) / 1e3, (tr[J][2] - (double)t0) / 1e3, (tr[J][3] - (double)t0) / 1e3,
             (tr[J][4] - (double)t0) / 1e3);
  return 0;
}
