// verify_div.cu — exhaustive/sampled proof that the forward's division
// shortcut is bit-identical to IEEE round-to-nearest division.
//
// The fused forward replaces z = x / s (IEEE, per element: MUFU.RCP + FFMA
// refinement + FCHK slow-path branch) by the Markstein-corrected quotient
//     y = RN(1/s) (once per vector unit), q0 = RN(x*y),
//     r = fma(-s, q0, x), z = fma(r, y, q0)
// guarded to |q0| < 2^100 and s in [2^-100, 2^100].
//
//  Test 1 (PROOF by exhaustion): for ALL 2^23 x 2^23 significand pairs
//    (x, s in [1, 2)), z == __fdiv_rn(x, s) bit for bit. In the normal
//    range every operation scales exactly by powers of two, so this covers
//    every normal x and s whose quotient is normal.
//  Test 2: for ALL 2^32 bit patterns x and a set of scales (random
//    log-uniform in [1e-6, 64], specials, all-ones significands), the full
//    FQ result of the fast path equals the IEEE-division FQ (covers zeros,
//    subnormals, infinities, NaN, overflow and underflow regions).
//  Test 2b: within test 2, every x passing the f32 screen |x| < s * 2^100
//    also through fq_value_fast_finite (negated residual, no guard, no
//    copysign) and fq_code_bits_fast_finite (int8 code), against IEEE.
//  Test 3 (evidence only): the double analogue with float numerators.
//
// Build/run (GPU box):  nvcc -O3 -gencode arch=compute_100a,code=sm_100a \
//     tools/verify_div.cu -o /tmp/verify_div && /tmp/verify_div
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <cuda_runtime.h>

#include "../paper_2511_12653_b200/csrc/qfb_device.cuh"

using namespace qfb;

__device__ unsigned long long g_bad;
__device__ unsigned long long g_first[8];

__global__ void pairs_kernel(uint32_t ms_base, uint32_t n_ms) {
  // one thread per (s significand, x significand block of 2^13)
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t ms = ms_base + (uint32_t)(t >> 10);
  if ((t >> 10) >= n_ms) return;
  const uint32_t mx0 = (uint32_t)(t & 1023u) << 13;
  const float s = __uint_as_float(0x3f800000u | ms);
  const float y = __frcp_rn(s);
  unsigned long long bad = 0;
  for (uint32_t k = 0; k < 8192; ++k) {
    const float x = __uint_as_float(0x3f800000u | (mx0 + k));
    const float ref = __fdiv_rn(x, s);
    const float z = markstein_div(x, s, y);
    if (__float_as_uint(ref) != __float_as_uint(z)) {
      if (bad == 0) {
        const unsigned long long i = atomicAdd(&g_bad, 0ull);
        if (i < 8) g_first[i] = ((unsigned long long)ms << 32) | (mx0 + k);
      }
      ++bad;
    }
  }
  if (bad) atomicAdd(&g_bad, bad);
}

__global__ void fq_all_x_kernel(const float* scales, int ns, uint64_t base) {
  const uint64_t t = base + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t xb = (uint32_t)t;
  const float x = __uint_as_float(xb);
  unsigned long long bad = 0;
  for (int i = 0; i < ns; ++i) {
    const float s = scales[i];
    const float y = __frcp_rn(s);
    const float a = fq_value(x, s, 127.0f);
    const float b = fq_value_fast(x, s, y, 127.0f);
    if (__float_as_uint(a) != __float_as_uint(b)) ++bad;
    // test 2b: the screened f32 paths (|x| < s * 2^100): FQ value without
    // guards / copysign, and the int8 code bits
    if (fast_div_ok(s) && fabsf(x) < __fmul_rn(s, 0x1p100f)) {
      const float c = fq_value_fast_finite(x, s, y, 127.0f);
      if (__float_as_uint(a) != __float_as_uint(c)) ++bad;
      const uint32_t cb = fq_code_bits_fast_finite(x, s, y, 127.0f) & 0xffu;
      if (cb != (uint32_t)(uint8_t)fq_code(x, s, 127.0f)) ++bad;
    }
  }
  if (bad) {
    const unsigned long long i = atomicAdd(&g_bad, bad);
    if (i < 8) g_first[i] = xb;
  }
}

__global__ void double_kernel(const double* scales, int ns) {
  const uint32_t mx = blockIdx.x * blockDim.x + threadIdx.x;  // 2^23 significands
  const double x = (double)__uint_as_float(0x3f800000u | (mx & 0x7fffffu));
  unsigned long long bad = 0;
  for (int i = 0; i < ns; ++i) {
    const double s = scales[i];
    const double y = __drcp_rn(s);
    const double ref = __ddiv_rn(x, s);
    const double q0 = __dmul_rn(x, y);
    const double r = __fma_rn(-s, q0, x);
    const double z = __fma_rn(r, y, q0);
    if (__double_as_longlong(ref) != __double_as_longlong(z)) ++bad;
  }
  if (bad) atomicAdd(&g_bad, bad);
}

static unsigned long long read_bad() {
  unsigned long long b = 0;
  cudaMemcpyFromSymbol(&b, g_bad, sizeof b);
  return b;
}
static void reset_bad() {
  unsigned long long z = 0;
  cudaMemcpyToSymbol(g_bad, &z, sizeof z);
}

int main(int argc, char** argv) {
  const bool quick = argc > 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms_t = 0;

  // ---- Test 1: all significand pairs ----
  reset_bad();
  cudaEventRecord(e0);
  const uint32_t total_ms = quick ? (1u << 12) : (1u << 23);
  const uint32_t per_launch = 1u << 17;  // s significands per launch
  for (uint32_t b = 0; b < total_ms; b += per_launch) {
    const uint32_t n = (total_ms - b) < per_launch ? (total_ms - b) : per_launch;
    const uint64_t threads = (uint64_t)n << 10;
    pairs_kernel<<<(unsigned)(threads / 256), 256>>>(b, n);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms_t, e0, e1);
  const unsigned long long bad1 = read_bad();
  printf("test1 markstein float quotient: %s significand pairs = %.3e, mismatches = %llu (%.1f s)\n",
         quick ? "SAMPLED" : "ALL", (double)total_ms * 8388608.0, bad1, ms_t / 1000);
  if (bad1) {
    unsigned long long f[8];
    cudaMemcpyFromSymbol(f, g_first, sizeof f);
    for (int i = 0; i < 8; ++i) printf("  first bad: s_sig=%#llx x_sig=%#llx\n", f[i] >> 32, f[i] & 0xffffffffull);
  }

  // ---- Test 2: FQ over all 2^32 x ----
  const int NS = quick ? 8 : 192;
  float hs[192];
  srand(12345);
  int k = 0;
  const float specials[] = {1e-6f, 1e-4f, 0.0315f, 1.0f, 2.0f, 64.0f, 0.5f, 1.99999988f,
                            3.99999976f, 1.5f, 0.75f, 1e-3f, 0.1f, 0.01f, 63.9999962f, 7.0f};
  for (; k < 16 && k < NS; ++k) hs[k] = specials[k];
  for (; k < NS; ++k) {
    const double u = (double)rand() / RAND_MAX;
    hs[k] = (float)exp(log(1e-6) + u * (log(64.0) - log(1e-6)));
  }
  float* ds;
  cudaMalloc(&ds, sizeof hs);
  cudaMemcpy(ds, hs, sizeof hs, cudaMemcpyHostToDevice);
  reset_bad();
  cudaEventRecord(e0);
  const uint64_t chunk = 1ull << 30;
  for (uint64_t base = 0; base < (1ull << 32); base += chunk)
    fq_all_x_kernel<<<(unsigned)(chunk / 256), 256>>>(ds, NS, base);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms_t, e0, e1);
  const unsigned long long bad2 = read_bad();
  printf("test2 FQ fast (+2b: screened finite value and int8 code) vs IEEE: all 2^32 x patterns x %d scales, mismatches = %llu (%.1f s)\n", NS,
         bad2, ms_t / 1000);

  // ---- Test 3: double analogue (evidence) ----
  const int ND = quick ? 64 : 4096;
  double* hd = (double*)malloc(sizeof(double) * ND);
  for (int i = 0; i < ND; ++i) {
    unsigned long long m = ((unsigned long long)rand() << 31) ^ (unsigned long long)rand();
    m = (m << 22) ^ (unsigned long long)rand();
    if (i < 8) m = (1ull << 52) - 1 - i;  // all-ones significands
    const unsigned long long bits = 0x3ff0000000000000ull | (m & ((1ull << 52) - 1));
    memcpy(&hd[i], &bits, 8);
  }
  double* dd;
  cudaMalloc(&dd, sizeof(double) * ND);
  cudaMemcpy(dd, hd, sizeof(double) * ND, cudaMemcpyHostToDevice);
  reset_bad();
  cudaEventRecord(e0);
  double_kernel<<<(1u << 23) / 256, 256>>>(dd, ND);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms_t, e0, e1);
  printf("test3 markstein double (float numerators): all 2^23 x significands x %d s, mismatches = %llu (%.1f s)\n",
         ND, read_bad(), ms_t / 1000);
  // (the backward's double quotient is validated by tools/verify_ddiv2.cu)
  cudaError_t err = cudaGetLastError();
  printf("cuda: %s\n", cudaGetErrorString(err));
  return (bad1 || bad2 || err != cudaSuccess) ? 1 : 0;
}
