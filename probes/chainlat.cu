#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double quot_v(double y, double u, double r, bool& ok) {
  const double q0 = y * r;
  const double q = fma(r, fma(-u, q0, y), q0);
  const double rr = fma(-u, q, y);
  const long long qb = __double_as_longlong(q);
  const long long e = qb & 0x7ff0000000000000LL;
  const bool normal = e > (54LL << 52) && e < (0x7feLL << 52);
  double lim = fabs(u) * __longlong_as_double(e - (53LL << 52));
  const bool below = (rr < 0.0) != (u < 0.0);
  const bool pow2 = (qb & 0x000fffffffffffffLL) == 0;
  if (pow2 && below == (q > 0.0)) lim *= 0.5;
  const bool pzero = __double_as_longlong(y) == 0;
  ok = ok && (pzero || (normal && fabs(rr) < lim));
  return q;
}
template <int MODE>
__global__ void k(double* out, long long* cyc, double u, double r, int iters) {
  double x = 1.0 + threadIdx.x * 1e-3;
  bool ok = true;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    if (MODE == 0) { x = quot_v(x, u, r, ok); x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 1) { bool o2 = true; double q = quot_v(x, u, r, o2); if (!o2) q = x / u; x = fma(-q, 1e-3, x + 1.0); }
    if (MODE == 2) { x = x / u; x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 3) { x = quot_v(x, u, r, ok); x = __shfl_sync(0xffffffffu, x, 0); x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 4) { if ((threadIdx.x & 3) == 0) x = quot_v(x, u, r, ok); x = __shfl_sync(0xffffffffu, x, threadIdx.x & ~3); x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 5) { x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 6) { const double q0 = x * r; const double q = fma(r, fma(-u, q0, x), q0); x = __shfl_sync(0xffffffffu, q, threadIdx.x & ~3); x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 7) { double q = x; if ((threadIdx.x & 3) == 0) { const double q0 = x * r; q = fma(r, fma(-u, q0, x), q0); } x = __shfl_sync(0xffffffffu, q, threadIdx.x & ~3); x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 8) { double q = x / u; x = __shfl_sync(0xffffffffu, q, threadIdx.x & ~3); x = fma(-x, 1e-3, x + 1.0); }
    if (MODE == 9) { double q = x; if ((threadIdx.x & 3) == 0) q = x / u; x = __shfl_sync(0xffffffffu, q, threadIdx.x & ~3); x = fma(-x, 1e-3, x + 1.0); }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + ok;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int MODE> void run(double* o, long long* c, const char* nm) {
  long long h;
  for (int r = 0; r < 3; r++) k<MODE><<<1, 32>>>(o, c, 3.0, 1.0 / 3.0, 4096);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"chain\", \"variant\": \"%s\", \"cycles_per_iter\": %.1f}\n", nm, h / 4096.0);
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  run<5>(o, c, "fma+add");
  run<0>(o, c, "quot_v+fma+add");
  run<1>(o, c, "quot_v_inline_fallback+fma+add");
  run<2>(o, c, "div+fma+add");
  run<3>(o, c, "quot_v+shfl+fma+add");
  run<4>(o, c, "divergent quot_v+shfl+fma+add");
  run<6>(o, c, "markstein_nocheck+shfl+fma+add");
  run<7>(o, c, "divergent markstein_nocheck+shfl+fma+add");
  run<8>(o, c, "div+shfl+fma+add");
  run<9>(o, c, "divergent div+shfl+fma+add");
  return 0;
}
