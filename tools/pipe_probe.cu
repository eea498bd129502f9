// pipe_probe.cu — memory-pipeline probe for the backward's traffic shape
// (read x and up, write d_input: 12 B/elem f32 over 41,164,800 elements,
// one 480x640 frame's quant points). Diagnostic tool, not product code:
// isolates which pipeline structure moves these bytes at HBM speed.
//
//   regs      : register-pipelined ld.global.nc.v4 (4 units in flight), st.global.v4
//   sync<NS>  : TMA ring, thread 0 issues NS-1 chunks ahead, all threads
//               compute from smem, st.global.v4 from registers, __syncthreads
//   ws<NS,S>  : 1 producer warp + 8 consumer warps, full/done mbarriers;
//               S=0 consumers store d_input from registers (st.global.v4);
//               S=1 consumers write d_input into the stage, the producer
//               bulk-stores it (TMA) and waits for the read before refilling
// Tile bytes per array: 16 KB aligned chunks, or `tile` bytes (e.g. 9600)
// to mimic tree-node tiles.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o pipe_probe tools/pipe_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));           \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(d)),
               "l"(s), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(smem_u32(s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t par) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(par)
      : "memory");
  return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  while (!try_wait(b, par)) {
  }
}
__device__ __forceinline__ uint4 ldnc(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t dx1(uint32_t x, uint32_t u) {
  return fabsf(__uint_as_float(x)) < 1.0f ? u : (u & 0x80000000u);
}
__device__ __forceinline__ uint4 dx4(uint4 x, uint4 u) {
  return make_uint4(dx1(x.x, u.x), dx1(x.y, u.y), dx1(x.z, u.z), dx1(x.w, u.w));
}

// tiles: [t*tile, min((t+1)*tile, n)) bytes, round robin over the grid
struct Args {
  const char* x;
  const char* up;
  char* dx;
  uint64_t bytes;   // per array
  uint32_t tile;    // bytes per tile (multiple of 16)
  uint32_t ntiles;
};

__global__ void __launch_bounds__(256) k_regs(Args a) {
  const uint64_t units = a.bytes / 16;
  const uint64_t stride = (uint64_t)gridDim.x * 256 * 4;
  for (uint64_t base = (uint64_t)blockIdx.x * 1024 + threadIdx.x; base < units; base += stride) {
    uint4 rx[4], ru[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t u = base + k * 256;
      if (u < units) {
        rx[k] = ldnc(a.x + 16 * u);
        ru[k] = ldnc(a.up + 16 * u);
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t u = base + k * 256;
      if (u < units) *reinterpret_cast<uint4*>(a.dx + 16 * u) = dx4(rx[k], ru[k]);
    }
  }
}

template <int NS>
__global__ void __launch_bounds__(256) k_sync(Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[NS];
  const uint32_t T = a.tile;
  auto issue = [&](uint32_t t, int s) {
    const uint64_t b0 = (uint64_t)t * T;
    const uint32_t nb = (uint32_t)((a.bytes - b0) < T ? (a.bytes - b0) : T);
    fence_async();
    expect_tx(&bar[s], 2 * nb);
    g2s(sm + (size_t)s * 2 * T, a.x + b0, nb, &bar[s]);
    g2s(sm + (size_t)s * 2 * T + T, a.up + b0, nb, &bar[s]);
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_init();
    for (int s = 0; s < NS - 1; ++s) {
      const uint32_t t = blockIdx.x + s * gridDim.x;
      if (t < a.ntiles) issue(t, s);
    }
  }
  __syncthreads();
  uint32_t ph = 0;
  int it = 0;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
    const int s = it % NS;
    if (threadIdx.x == 0) {
      const uint32_t n = t + (NS - 1) * gridDim.x;
      if (n < a.ntiles) issue(n, (it + NS - 1) % NS);
    }
    wait(&bar[s], (ph >> s) & 1);
    ph ^= 1u << s;
    const uint64_t b0 = (uint64_t)t * T;
    const uint32_t nb = (uint32_t)((a.bytes - b0) < T ? (a.bytes - b0) : T);
    const uint4* sx = reinterpret_cast<const uint4*>(sm + (size_t)s * 2 * T);
    const uint4* su = reinterpret_cast<const uint4*>(sm + (size_t)s * 2 * T + T);
    for (uint32_t k = threadIdx.x; k < nb / 16; k += 256)
      *reinterpret_cast<uint4*>(a.dx + b0 + 16 * k) = dx4(sx[k], su[k]);
    __syncthreads();
  }
}

template <int NS, int S>
__global__ void __launch_bounds__(288) k_ws(Args a) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[NS], done[NS];
  const uint32_t T = a.tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], 8);
    }
    fence_init();
  }
  __syncthreads();
  if (warp == 8) {
    auto issue = [&](uint32_t t, int s) {
      const uint64_t b0 = (uint64_t)t * T;
      const uint32_t nb = (uint32_t)((a.bytes - b0) < T ? (a.bytes - b0) : T);
      fence_async();
      expect_tx(&full[s], 2 * nb);
      g2s(sm + (size_t)s * 2 * T, a.x + b0, nb, &full[s]);
      g2s(sm + (size_t)s * 2 * T + T, a.up + b0, nb, &full[s]);
    };
    if (lane == 0) {
      for (int s = 0; s < NS; ++s) {
        const uint32_t t = blockIdx.x + s * gridDim.x;
        if (t < a.ntiles) issue(t, s);
      }
      uint32_t ph = 0;
      int s = 0;
      for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        wait(&done[s], (ph >> s) & 1);
        ph ^= 1u << s;
        if (S == 1) {
          const uint64_t b0 = (uint64_t)t * T;
          const uint32_t nb = (uint32_t)((a.bytes - b0) < T ? (a.bytes - b0) : T);
          s2g(a.dx + b0, sm + (size_t)s * 2 * T, nb);
          commit();
          wait_read();
        }
        const uint32_t n = t + NS * gridDim.x;
        if (n < a.ntiles) issue(n, s);
        s = s + 1 == NS ? 0 : s + 1;
      }
      wait_all();
    }
    return;
  }
  uint32_t ph = 0;
  int s = 0;
  for (uint32_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    wait(&full[s], (ph >> s) & 1);
    ph ^= 1u << s;
    const uint64_t b0 = (uint64_t)t * T;
    const uint32_t nb = (uint32_t)((a.bytes - b0) < T ? (a.bytes - b0) : T);
    uint4* sx = reinterpret_cast<uint4*>(sm + (size_t)s * 2 * T);
    const uint4* su = reinterpret_cast<const uint4*>(sm + (size_t)s * 2 * T + T);
    for (uint32_t k = threadIdx.x; k < nb / 16; k += 256) {
      const uint4 d = dx4(sx[k], su[k]);
      if (S == 1) sx[k] = d;
      else *reinterpret_cast<uint4*>(a.dx + b0 + 16 * k) = d;
    }
    if (S == 1) fence_async();
    __syncwarp();
    if (lane == 0) arrive(&done[s]);
    s = s + 1 == NS ? 0 : s + 1;
  }
}

template <typename K>
float run(K kern, int threads, size_t smem, Args a, int ctas_per_sm, int reps, int* occ_out) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  *occ_out = occ;
  const int per = ctas_per_sm < occ ? ctas_per_sm : occ;
  if (per < 1) return -1.f;
  const int grid = sms * per;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) kern<<<grid, threads, smem>>>(a);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) kern<<<grid, threads, smem>>>(a);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaGetLastError());
  return ms / reps * 1000.f;
}

int main(int argc, char** argv) {
  const uint64_t n = 41164800ull;
  const uint64_t bytes = n * 4;
  char *x, *up, *dx;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMalloc(&up, bytes));
  CK(cudaMalloc(&dx, bytes));
  CK(cudaMemset(x, 0x3e, bytes));
  CK(cudaMemset(up, 0x3f, bytes));
  const double alg = 3.0 * bytes;
  auto report = [&](const char* name, uint32_t tile, int per, float us, int occ) {
    printf("%-14s tile %6u  ctas/sm %d (occ %d)  %8.2f us  %7.1f GB/s\n", name, tile, per, occ, us,
           us > 0 ? alg / (us * 1e3) : 0.0);
  };
  const int reps = 20;
  for (uint32_t tile : {16384u, 9600u, 8192u, 32768u}) {
    Args a{x, up, dx, bytes, tile, (uint32_t)((bytes + tile - 1) / tile)};
    int occ;
    float us;
    if (tile == 16384u) {
      for (int per : {2, 4, 8}) {
        us = run(k_regs, 256, 0, a, per, reps, &occ);
        report("regs", tile, per, us, occ);
      }
    }
    for (int per : {2, 3, 4}) {
      us = run(k_sync<2>, 256, 2 * 2 * (size_t)tile, a, per, reps, &occ);
      report("sync<2>", tile, per, us, occ);
      us = run(k_sync<3>, 256, 3 * 2 * (size_t)tile, a, per, reps, &occ);
      report("sync<3>", tile, per, us, occ);
      us = run(k_ws<2, 0>, 288, 2 * 2 * (size_t)tile, a, per, reps, &occ);
      report("ws<2,reg>", tile, per, us, occ);
      us = run(k_ws<3, 0>, 288, 3 * 2 * (size_t)tile, a, per, reps, &occ);
      report("ws<3,reg>", tile, per, us, occ);
      us = run(k_ws<2, 1>, 288, 2 * 2 * (size_t)tile, a, per, reps, &occ);
      report("ws<2,bulk>", tile, per, us, occ);
      us = run(k_ws<3, 1>, 288, 3 * 2 * (size_t)tile, a, per, reps, &occ);
      report("ws<3,bulk>", tile, per, us, occ);
    }
  }
  return 0;
}
