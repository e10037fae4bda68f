// Probe: what bounds a one-thread-per-row elimination chain (64 steps, the
// row's entries in registers, the U rows broadcast from shared memory) on
// sm_100a.  Variants: full step (verified quotient + 63-k fma from shared U),
// no quotient (multiply), U from registers (no shared loads), and warps per
// CTA.  Output: cycles per step (%clock64 of thread 0).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
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

template <int MODE, int NW>
__global__ void __launch_bounds__(NW * 32) chain(double* out, long long* cyc, const double* U) {
  constexpr int W = 64;
  __shared__ __align__(16) double sU[W * W + W];
  __shared__ double sR[W];
  __shared__ __align__(8) uint64_t bar[W];
  for (int i = threadIdx.x; i < W * W; i += blockDim.x) sU[i] = U[i] + (i % 65 == 0 ? 2.0 : 0.0);
  for (int k = threadIdx.x; k < W; k += blockDim.x) sR[k] = 0.5;
  if (threadIdx.x == 0) {
    for (int k = 0; k < W; k++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  for (int k = threadIdx.x; k < W; k += blockDim.x)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&bar[k])) : "memory");
  __syncthreads();
  bool okall = true;
  double x[W];
#pragma unroll
  for (int c = 0; c < W; c++) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  const long long t0 = clock64();
#pragma unroll 1
  for (int rep = 0; rep < 4; rep++) {
#pragma unroll 1
    for (int qk = 0; qk < 8; qk++) {
#pragma unroll
      for (int o = 0; o < 8; o++) {
        const int k = qk * 8 + o;
        const double* uk = sU + k * W + 8 * qk;
        double l;
        if (MODE == 4 || MODE == 5) {
          uint32_t done;
          do {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(smem_addr(&bar[k])) : "memory");
          } while (!done);
        }
        if (MODE == 2) l = x[o] * 0.999;
        else if (MODE == 3 || MODE == 5) {
          bool ok = true;
          l = quot_v(x[o], uk[o], sR[k], ok);
          if (!ok) l = x[o] / uk[o];
        }
        else l = x[o] * uk[o];
        x[o] = l;
#pragma unroll
        for (int c = o + 1; c < W; c++) {
          const double u = (MODE == 2) ? 1e-3 * c : uk[c];
          x[c] = fma(-l, u, x[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < W - 8; c++) x[c] = x[c + 8] * (MODE == 3 ? 1.0 : 1.0);
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < W; c++) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// rotation by one per step: x[0] is always the current column; the fma for
// column c writes slot c - 1 (the shift costs no moves); U rows left-aligned
template <int NW, bool QUOT>
__global__ void __launch_bounds__(NW * 32) chain1(double* out, long long* cyc, const double* U) {
  constexpr int W = 64;
  __shared__ __align__(16) double sU[W * W];
  __shared__ double sR[W];
  for (int i = threadIdx.x; i < W * W; i += blockDim.x) sU[i] = U[i] + (i % 64 == 0 ? 2.0 : 0.0);
  for (int k = threadIdx.x; k < W; k += blockDim.x) sR[k] = 0.5;
  __syncthreads();
  double x[W];
#pragma unroll
  for (int c = 0; c < W; c++) x[c] = 1.0 + 1e-3 * (threadIdx.x + c);
  bool ok = true;
  double acc = 0;
  const long long t0 = clock64();
#pragma unroll 1
  for (int rep = 0; rep < 4; rep++) {
#pragma unroll 1
    for (int k = 0; k < W; k++) {
      const double* uk = sU + k * W;
      double l;
      if (QUOT) l = quot_v(x[0], uk[0], sR[k], ok);
      else l = x[0] * uk[0];
      acc += l;
#pragma unroll
      for (int c = 1; c < W; c += 2) {
        const double2 u2 = *reinterpret_cast<const double2*>(uk + c - 1);
        if (c > 1) x[c - 2] = fma(-l, u2.x, x[c - 1]);
        x[c - 1] = fma(-l, u2.y, x[c]);
      }
      x[W - 2] = fma(-l, uk[W - 1], x[W - 1]);
      x[W - 1] = 0.0;
    }
  }
  const long long t1 = clock64();
  double s = acc + (ok ? 0.0 : 1.0);
#pragma unroll
  for (int c = 0; c < W; c++) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int NW, bool QUOT>
void run1(double* out, long long* cyc, const double* U, const char* name) {
  long long h;
  for (int r = 0; r < 2; r++) chain1<NW, QUOT><<<1, NW * 32>>>(out, cyc, U);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"rowchain\", \"variant\": \"%s\", \"warps\": %d, \"cycles_per_step\": %.1f}\n", name, NW, h / 256.0);
}

template <int MODE, int NW>
void run(double* out, long long* cyc, const double* U, const char* name) {
  long long h;
  for (int r = 0; r < 2; r++) chain<MODE, NW><<<1, NW * 32>>>(out, cyc, U);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  chain<MODE, NW><<<1, NW * 32>>>(out, cyc, U);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"probe\": \"rowchain\", \"variant\": \"%s\", \"warps\": %d, \"cycles_per_step\": %.1f, \"ns_per_step\": %.1f}\n",
         name, NW, h / 256.0, ms * 1e6 / 256.0);
}

int main() {
  double *out, *U; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&U, 64 * 64 * 8); cudaMalloc(&cyc, 8);
  cudaMemset(U, 0, 64 * 64 * 8);
  run1<1, false>(out, cyc, U, "rot1");
  run1<2, false>(out, cyc, U, "rot1");
  run1<4, false>(out, cyc, U, "rot1");
  run1<1, true>(out, cyc, U, "rot1+quot");
  run1<2, true>(out, cyc, U, "rot1+quot");
  run1<4, true>(out, cyc, U, "rot1+quot");
  run<0, 1>(out, cyc, U, "smem_u");
  run<0, 4>(out, cyc, U, "smem_u");
  run<0, 8>(out, cyc, U, "smem_u");
  run<3, 4>(out, cyc, U, "smem_u+quot");
  run<4, 4>(out, cyc, U, "smem_u+wait");
  run<5, 4>(out, cyc, U, "smem_u+quot+wait");
  run<5, 1>(out, cyc, U, "smem_u+quot+wait");
  run<2, 1>(out, cyc, U, "reg_u");
  run<2, 4>(out, cyc, U, "reg_u");
  run<2, 8>(out, cyc, U, "reg_u");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
