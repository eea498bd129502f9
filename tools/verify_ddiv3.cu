// verify_ddiv3.cu — validation of the backward's double quotient with a
// double-double reciprocal and ONE Markstein correction:
//     y = RN(1/s); y_lo = RN(RN(1 - s*y) * y)   (per tile; 1 - s*y is exact)
//     q0 = RN(x*y + RN(x*y_lo))                 (fma)
//     z  = RN(q0 + (x - s*q0)*y)                (fma; the residual is exact)
// y + y_lo = (1/s)(1 + d), |d| <= ~2^-105, and RN(x*y_lo) errs by at most
// 2^-106 |x*y|, so q0 lies within 1/2 ulp + 2^-103 |x/s| of x/s: faithful.
// Markstein's theorem (y = RN(1/s), q0 faithful) makes z = RN(x/s). Four
// FP64 ops (DMUL + 3 DFMA, dependency depth 4) instead of five (depth 5) in
// markstein2_div. This tool checks it against __ddiv_rn for EVERY finite
// float x (2^32 patterns, zeros included) and the scale set of
// verify_ddiv2.cu (random log-uniform over [2^-100, 2^100], the DPVO range
// [1e-6, 64], adversarial significands), plus non-finite x -> NaN.
//
// Build/run (GPU box):  nvcc -O3 -gencode arch=compute_100a,code=sm_100a \
//     tools/verify_ddiv3.cu -o /tmp/verify_ddiv3 && /tmp/verify_ddiv3 [n_random]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

__device__ unsigned long long g_bad;
__device__ unsigned long long g_first[8];

__device__ int g_single;  // 1: control = ONE correction from q0 = RN(x*y) (no y_lo)

__device__ __forceinline__ double ddiv2(double x, double s, double y, double ylo) {
  const double q0 = g_single ? __dmul_rn(x, y) : __fma_rn(x, y, __dmul_rn(x, ylo));
  return __fma_rn(__fma_rn(-s, q0, x), y, q0);
}
__device__ __forceinline__ double recip_lo(double s, double y) { return __dmul_rn(__fma_rn(-s, y, 1.0), y); }

__global__ void all_x_kernel(const double* scales, int ns) {
  const int si = blockIdx.y;
  if (si >= ns) return;
  const double s = scales[si];
  const double y = __drcp_rn(s);
  const double ylo = recip_lo(s, y);
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;  // 2^20 threads
  unsigned long long bad = 0;
  for (uint32_t k = 0; k < 4096; ++k) {
    const uint32_t bits = (uint32_t)(t * 4096u + k);
    const float xf = __uint_as_float(bits);
    const double x = (double)xf;
    const double z = ddiv2(x, s, y, ylo);
    bool ok;
    if (!isfinite(xf)) {
      ok = isnan(z);  // inf/NaN x: the fast path needs NaN (mask false)
    } else if (xf == 0.0f) {
      ok = z == 0.0;  // +-0: a zero (its sign is not observed: rint(z) - z = +0)
    } else {
      ok = __double_as_longlong(__ddiv_rn(x, s)) == __double_as_longlong(z);
    }
    if (!ok) {
      const unsigned long long i = atomicAdd(&g_bad, 1ull);
      if (i < 8) g_first[i] = ((unsigned long long)si << 32) | bits;
      ++bad;
    }
  }
}

// Random double numerators (53-bit significands, exponents within +-60 of
// the divisor's) against the same divisors: the distillation loss divides
// doubles (2d/n, b/nrm, cos*a/na2) with hoisted reciprocals too.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__global__ void random_num_kernel(const double* scales, int ns, uint32_t per_thread) {
  const int si = blockIdx.y;
  if (si >= ns) return;
  const double s = scales[si];
  const double y = __drcp_rn(s);
  const double ylo = recip_lo(s, y);
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int es = (int)((__double_as_longlong(s) >> 52) & 0x7ff);
  for (uint32_t k = 0; k < per_thread; ++k) {
    const uint64_t r = mix64((t << 20) ^ ((uint64_t)si << 44) ^ k);
    int e = es + (int)((r >> 52) % 121) - 60;
    if (e < 200) e = 200;  // keep quotients and residuals normal (well inside the range)
    if (e > 1800) e = 1800;
    const double x = __longlong_as_double((long long)((r & 0x800fffffffffffffull) | ((uint64_t)e << 52)));
    if (__double_as_longlong(__ddiv_rn(x, s)) != __double_as_longlong(ddiv2(x, s, y, ylo))) {
      const unsigned long long i = atomicAdd(&g_bad, 1ull);
      if (i < 8) g_first[i] = ((unsigned long long)si << 32) | k;
    }
  }
}

int main(int argc, char** argv) {
  const int n_random = argc > 1 ? atoi(argv[1]) : 2048;
  const int single = argc > 2 ? atoi(argv[2]) : 0;
  cudaMemcpyToSymbol(g_single, &single, sizeof single);
  std::vector<double> sc;
  std::mt19937_64 rng(2511);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  for (int i = 0; i < n_random; ++i) sc.push_back(std::ldexp(1.0 + u(rng), (int)std::floor(-100 + 200 * u(rng))));
  for (int i = 0; i < n_random; ++i) sc.push_back(std::exp(std::log(1e-6) + (std::log(64.0) - std::log(1e-6)) * u(rng)));
  for (int e = -100; e < 100; e += 7) {
    sc.push_back(std::ldexp(1.0, e));                               // powers of two
    sc.push_back(std::ldexp(2.0 - std::ldexp(1.0, -52), e));        // all-ones significand
    for (int k = 1; k < 4; ++k) sc.push_back(std::ldexp(1.0 + k * std::ldexp(1.0, -52), e));
    sc.push_back(std::ldexp(1.5, e));
    sc.push_back(std::ldexp(1.0 + std::ldexp(1.0, -26), e));
    sc.push_back(std::ldexp(2.0 - std::ldexp(1.0, -26), e));
    sc.push_back(std::ldexp(std::sqrt(2.0), e));
    sc.push_back(std::ldexp(1.0 / 3.0 * 2.0, e));
  }
  const int ns = (int)sc.size();
  double* d_sc;
  cudaMalloc(&d_sc, ns * sizeof(double));
  cudaMemcpy(d_sc, sc.data(), ns * sizeof(double), cudaMemcpyHostToDevice);
  const unsigned long long zero = 0;
  cudaMemcpyToSymbol(g_bad, &zero, sizeof zero);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int chunk = 64;
  for (int b = 0; b < ns; b += chunk) {
    const int n = ns - b < chunk ? ns - b : chunk;
    all_x_kernel<<<dim3((1u << 20) / 256, n), 256>>>(d_sc + b, n);
  }
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  // double numerators: 2^30 random per scale
  unsigned long long bad_f = 0;
  cudaMemcpyFromSymbol(&bad_f, g_bad, sizeof bad_f);
  cudaEventRecord(e0);
  for (int b = 0; b < ns; b += chunk) {
    const int n = ns - b < chunk ? ns - b : chunk;
    random_num_kernel<<<dim3((1u << 20) / 256, n), 256>>>(d_sc + b, n, 1024);
  }
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms2 = 0;
  cudaEventElapsedTime(&ms2, e0, e1);
  unsigned long long bad_all = 0;
  cudaMemcpyFromSymbol(&bad_all, g_bad, sizeof bad_all);
  printf("verify_ddiv3 double numerators: %d scales x 2^30 random doubles: %llu mismatches (%.1f s)\n", ns,
         bad_all - bad_f, ms2 / 1e3);
  unsigned long long bad = 0, first[8];
  cudaMemcpyFromSymbol(&bad, g_bad, sizeof bad);
  cudaMemcpyFromSymbol(first, g_first, sizeof first);
  printf("verify_ddiv3%s: %s; %d scales x all 2^32 float x (finite: bitwise; 0: zero; inf/NaN: NaN): %llu mismatches vs __ddiv_rn "
         "(%.1f s)\n", single ? " [control: no y_lo]" : "", cudaGetErrorString(err), ns, bad, ms / 1e3);
  for (unsigned long long i = 0; i < bad && i < 8; ++i)
    printf("  scale %.17g x bits 0x%08x\n", sc[first[i] >> 32], (unsigned)(first[i] & 0xffffffffu));
  return (single || bad == 0) && err == cudaSuccess ? 0 : 1;
}
