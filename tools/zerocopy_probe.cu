// zerocopy_probe.cu — PCIe throughput of kernels that read / write pinned
// host memory directly (no DMA copies), one DPVO frame's worth of bytes per
// direction, each alone and both at once; compared with cudaMemcpyAsync.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/zerocopy_probe.cu -o /tmp/zc && /tmp/zc
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n) v[k] = src[i + k * stride];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * stride < n) dst[i + k * stride] = v[k];
  }
}

int main() {
  const size_t in_b = 305971200, out_b = 329325616 & ~size_t(15);
  void *h_in, *h_out, *d_in, *d_out;
  cudaMallocHost(&h_in, in_b);
  cudaMallocHost(&h_out, out_b);
  cudaMalloc(&d_in, in_b);
  cudaMalloc(&d_out, out_b);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, int mode, int blocks_per_sm) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      if (mode & 1) copy_kernel<<<sms * blocks_per_sm, 256, 0, s1>>>((const uint4*)h_in, (uint4*)d_in, in_b / 16);
      if (mode & 2) copy_kernel<<<sms * blocks_per_sm, 256, 0, s2>>>((const uint4*)d_out, (uint4*)h_out, out_b / 16);
      if (mode & 4) cudaMemcpyAsync(d_in, h_in, in_b, cudaMemcpyHostToDevice, s1);
      if (mode & 8) cudaMemcpyAsync(h_out, d_out, out_b, cudaMemcpyDeviceToHost, s2);
      cudaStreamSynchronize(s1);
      cudaStreamSynchronize(s2);
      cudaEventRecord(e1, 0);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1) printf("%-34s %8.3f ms\n", name, ms);
    }
  };
  run("dma h2d", 4, 1);
  run("dma d2h", 8, 1);
  run("dma both", 12, 1);
  for (int b : {1, 2, 4}) {
    char n1[64], n2[64], n3[64];
    snprintf(n1, 64, "kernel h2d (%d CTA/SM)", b);
    snprintf(n2, 64, "kernel d2h (%d CTA/SM)", b);
    snprintf(n3, 64, "kernel both (%d+%d CTA/SM)", b, b);
    run(n1, 1, b);
    run(n2, 2, b);
    run(n3, 3, b);
  }
  printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
