// fp64_probe.cu — per-instruction throughput of the backward's arithmetic on
// this GPU (diagnostic tool, not product code): DFMA, DADD, FRND.F64 (rint),
// F2F.F64.F32 (float -> double), F2F.F64.F16, DSETP, and the integer-ALU
// float->double widening. Each kernel runs 8 independent chains per thread
// over a long loop; results are ops per clock per SM at the SM clock
// measured with clock64().
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o fp64_probe tools/fp64_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kIters = 4096;
constexpr int kChains = 8;

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ unsigned long long g_cycles[1024];

template <int OP>
__global__ void probe(double* out, float seed) {
  double d[kChains];
  float f[kChains];
  __half h[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    f[c] = seed + threadIdx.x * 1e-3f + c;
    d[c] = (double)f[c];
    h[c] = __float2half(f[c]);
  }
  const long long t0 = clock64();
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      if constexpr (OP == 0) d[c] = fma(d[c], 1.0000001, 1e-9);              // DFMA
      if constexpr (OP == 1) d[c] = d[c] + 1e-9;                             // DADD
      if constexpr (OP == 2) d[c] = rint(d[c]) + 0.25;                        // FRND.F64 + DADD
      if constexpr (OP == 3) {                                                // F2F.F64.F32 (+ FADD to vary)
        d[c] += (double)f[c];
        f[c] = f[c] + 1.0f;
      }
      if constexpr (OP == 4) {                                                // F2F.F64.F16
        double v;
        asm volatile("cvt.f64.f16 %0, %1;" : "=d"(v) : "h"(__half_as_ushort(h[c])));
        d[c] += v;
        h[c] = __hadd(h[c], __float2half(1.0f));
      }
      if constexpr (OP == 5) {                                                // integer widening of a normal float
        const unsigned b = __float_as_uint(f[c]);
        const unsigned hi = (b & 0x80000000u) | (((b >> 3) & 0x0fffffffu) + 0x38000000u);
        d[c] += __hiloint2double((int)hi, (int)(b << 29));
        f[c] = f[c] + 1.0f;
      }
      if constexpr (OP == 6) d[c] = rint(d[c]) * 1.5;                         // FRND.F64 + DMUL
    }
  }
  const long long t1 = clock64();
  double acc = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc += d[c] + (double)f[c] + (double)__half2float(h[c]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int threads = 512, blocks = sms * 2;
  double* out;
  CK(cudaMalloc(&out, (size_t)blocks * threads * sizeof(double)));
  const char* names[] = {"DFMA", "DADD", "FRND.F64+DADD", "F2F.F64.F32+DADD(+FADD)", "F2F.F64.F16+DADD(+HADD)",
                         "int-widen+DADD(+FADD)", "FRND.F64+DMUL"};
  for (int op = 0; op < 7; ++op) {
    auto launch = [&] {
      switch (op) {
        case 0: probe<0><<<blocks, threads>>>(out, 1.5f); break;
        case 1: probe<1><<<blocks, threads>>>(out, 1.5f); break;
        case 2: probe<2><<<blocks, threads>>>(out, 1.5f); break;
        case 3: probe<3><<<blocks, threads>>>(out, 1.5f); break;
        case 4: probe<4><<<blocks, threads>>>(out, 1.5f); break;
        case 5: probe<5><<<blocks, threads>>>(out, 1.5f); break;
        default: probe<6><<<blocks, threads>>>(out, 1.5f); break;
      }
    };
    launch();
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc[1024];
    CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * blocks));
    double avg = 0;
    for (int i = 0; i < blocks; ++i) avg += (double)cyc[i];
    avg /= blocks;
    // 2 blocks per SM resident together: ops per SM = 2 * threads * iters * chains
    const double ops_per_sm = 2.0 * threads * (double)kIters * kChains;
    printf("%-28s %8.1f ops/clk/SM (loop %.0f cycles)  %.3f ms  %.2f Tops/s\n", names[op], ops_per_sm / avg, avg, ms,
           (double)blocks * threads * kIters * kChains / (ms * 1e-3) / 1e12);
  }
  return 0;
}
