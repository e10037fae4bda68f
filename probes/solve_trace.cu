// Probe: timeline of the wavefront solve (per row block: start, last-tile
// wait begin/end, diagonal begin, diagonal end, release) via %globaltimer.
#define EBV_SOLVE_TRACE 1
#include "../paper_1907_05767_b200/csrc/k_solve.cu"
#include <cstdio>
#include <vector>
#include <random>
int main(int argc, char** argv) {
  int64_t n = argc > 1 ? atoll(argv[1]) : 32768;
  int nrhs = argc > 2 ? atoi(argv[2]) : 1;
  std::vector<double> hLU((size_t)n * n);
  std::mt19937_64 rng(1);
  std::uniform_real_distribution<double> u(-1e-3, 1e-3);
  for (int64_t j = 0; j < n; j++)
    for (int64_t i = 0; i < n; i++) hLU[i + j * n] = (i == j) ? 1.0 + u(rng) : u(rng) / n;
  double *dLU, *dB;
  int *ticket, *flags;
  cudaMalloc(&dLU, (size_t)n * n * 8);
  cudaMalloc(&dB, (size_t)n * nrhs * 8);
  cudaMalloc(&ticket, 8);
  cudaMalloc(&flags, 128 * ((n + 63) / 64) * 4);
  cudaMemset(flags, 0, 128 * ((n + 63) / 64) * 4);
  cudaMemcpy(dLU, hLU.data(), (size_t)n * n * 8, cudaMemcpyHostToDevice);
  std::vector<double> hB((size_t)n * nrhs, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 1; rep <= 3; rep++) {
    cudaMemcpy(dB, hB.data(), hB.size() * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    ebv::launch_solve(n, dLU, n, dB, n, nrhs, ticket, flags, rep, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("rep %d solve %.3f ms (err %s)\n", rep, ms, cudaGetErrorString(cudaGetLastError()));
  }
  static unsigned long long tr[2][8192][6];
  cudaMemcpyFromSymbol(tr, ebv::g_trace, sizeof(tr));
  int redo = 0;
  cudaMemcpyFromSymbol(&redo, ebv::g_redo, sizeof(int));
  printf("backward blocks redone with true division (all reps, per warp): %d\n", redo);
  int64_t NB = (n + 63) / 64;
  for (int d = 0; d < 2; d++) {
    unsigned long long t0 = ~0ull;
    for (int64_t I = 0; I < NB; I++) t0 = tr[d][I][0] < t0 ? tr[d][I][0] : t0;
    printf("%s: block start(us) lastwait_begin lastwait_end diag_begin diag_end release\n", d ? "backward" : "forward");
    for (int64_t I = 0; I < NB; I++) {
      int64_t J = d ? NB - 1 - I : I;
      if (I < 6 || I % (NB / 16 > 0 ? NB / 16 : 1) == 0 || I > NB - 4)
        printf("  %5lld: %9.2f %9.2f %9.2f %9.2f %9.2f %9.2f\n", (long long)J, (tr[d][J][0] - t0) / 1e3,
               (tr[d][J][1] - t0) / 1e3, (tr[d][J][2] - t0) / 1e3, (tr[d][J][3] - t0) / 1e3, (tr[d][J][4] - t0) / 1e3,
               (tr[d][J][5] - t0) / 1e3);
    }
  }
  return 0;
}
