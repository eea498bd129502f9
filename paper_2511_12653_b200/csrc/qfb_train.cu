// qfb_train.cu — the on-device pieces of the scale-only QAT step around the
// fake-quant path, bit-exact with the reference:
//
//  - distillation loss per tensor pair (distill.hpp:66-124 pair_loss): MSE
//    over all elements with the fixed pairwise tree (tensor.hpp:100-109),
//    per-location cosine over the channel axis (sequential channel folds in
//    double, zero-norm locations guarded), and the student gradient
//    d_s = float(2d/n) (+)= float(-w (b/nrm - cos a/na2)) in float32, then the
//    trainer's chunk scaling float(d * inv) (distill.hpp:243-246);
//  - Adam over the flattened scale vector (distill.hpp:264-279) with the
//    trainer's skip rule (a non-finite gradient skips the whole update,
//    distill.hpp:254-258), decided on the device so the step stays
//    capturable in a CUDA graph.
//
// The exact pairwise sum of n terms runs as: one thread per leaf group of
// the reference tree (depth D = least with ceil(n/2^D) <= 16; a group is
// fold(first half) + fold(second half) from 0.0, or one fold if <= 8), then
// perfect-tree halving of the 2^D group sums in shared memory, 2048 per CTA
// per pass (the tree above depth D is perfect). All HBM
// traffic is one read of s and t, one write of d_s: the loss is HBM-bound.
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/qfb.h"
#include "qfb_device.cuh"
#include "qfb_kernels.h"

namespace qfb {
namespace {

constexpr int kLeaf = 16;
constexpr int kRedThreads = 1024;  // halving kernel: 2048 values per CTA

__host__ __device__ __forceinline__ uint32_t tree_depth(uint64_t n) {
  uint32_t d = 0;
  while (((n + (1ull << d) - 1) >> d) > (uint64_t)kLeaf) ++d;
  return d;
}

// Node `g` at depth `levels` of the reference split of [0, n).
__device__ __forceinline__ void node_of(uint64_t n, uint32_t g, uint32_t levels, uint64_t& lo,
                                        uint64_t& m) {
  lo = 0;
  m = n;
  for (int l = (int)levels - 1; l >= 0; --l) {
    const uint64_t h = m >> 1;
    if ((g >> l) & 1u) {
      lo += h;
      m -= h;
    } else {
      m = h;
    }
  }
}

// MSE terms of pair_loss (distill.hpp:84-91): d = double(s) - double(t),
// term d*d (the matching gradient 0.0f + float(2d/n) is produced by the
// cosine kernel, which reads s and t anyway).
__device__ __forceinline__ double mse_term(float sv, float tv) {
  const double d = __dadd_rn((double)sv, -(double)tv);
  return __dmul_rn(d, d);
}

// Stored terms (cosines per location).
struct LoadTerm {
  const double* v;
  uint64_t stride;
  __device__ __forceinline__ double operator()(uint32_t b, uint64_t i) const {
    return v[(uint64_t)b * stride + i];
  }
};

template <typename Term>
__device__ __forceinline__ double fold(const Term& f, uint32_t b, uint64_t lo, uint64_t m) {
  double acc = 0.0;
  for (uint64_t k = 0; k < m; ++k) acc = __dadd_rn(acc, f(b, lo + k));
  return acc;
}

// One thread per leaf group of pair b = blockIdx.y: its sum in the
// reference order.
template <typename Term>
__global__ void leaf_sums_kernel(Term f, uint64_t n, uint32_t depth, double* out) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t b = blockIdx.y;
  if (g >= (1u << depth)) return;
  uint64_t lo, m;
  node_of(n, g, depth, lo, m);
  double r;
  if (m <= 8) {
    r = fold(f, b, lo, m);
  } else {
    const uint64_t h = m >> 1;
    r = __dadd_rn(fold(f, b, lo, h), fold(f, b, lo + h, m - h));
  }
  out[((uint64_t)b << depth) + g] = r;
}

// MSE leaf sums with coalesced loads: warp w of a CTA owns 32 consecutive
// leaf groups (<= 512 contiguous elements), stages their s and t through
// shared memory with 16-byte loads (scalar when the pointers are not
// 16-byte aligned), then each lane folds its group in the reference order.
// With kSub, the CTA's 256 groups — an aligned perfect subtree — are
// reduced to one value (warp xor butterfly, then the 8 warp sums as a
// perfect tree) so only 2^(depth-8) values per pair go to the halving
// passes. Pair b = blockIdx.y.
constexpr int kMseWarps = 8;
constexpr int kMseSubLog = 8;  // log2(32 * kMseWarps)
template <bool kSub>
__global__ void __launch_bounds__(kMseWarps * 32) mse_leaf_kernel(const float* __restrict__ s,
                                                                 const float* __restrict__ t, uint64_t n,
                                                                 uint32_t depth, double* out) {
  __shared__ __align__(16) float ss[kMseWarps][2][32 * kLeaf + 8];
  __shared__ double wsum[kMseWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t b = blockIdx.y;
  const uint32_t groups = 1u << depth;
  const uint32_t g = (blockIdx.x * kMseWarps + warp) * 32u + (uint32_t)lane;
  uint64_t lo = 0, m = 0;
  if (g < groups) {
    if (n < (1ull << 32)) {  // the descent in 32-bit arithmetic (same values)
      uint32_t lo32 = 0, m32 = (uint32_t)n;
      for (int l = (int)depth - 1; l >= 0; --l) {
        const uint32_t h = m32 >> 1;
        const bool right = (g >> l) & 1u;
        lo32 += right ? h : 0u;
        m32 = right ? m32 - h : h;
      }
      lo = lo32;
      m = m32;
    } else {
      node_of(n, g, depth, lo, m);
    }
  }
  // the warp's element range [w0, w1)
  const uint64_t w0 = __shfl_sync(0xffffffffu, lo, 0);
  const uint32_t last = min(31u, groups > (g - lane) ? groups - (g - lane) - 1u : 0u);
  const uint64_t w1 = __shfl_sync(0xffffffffu, lo + m, (int)last);
  if (g - (uint32_t)lane >= groups) return;  // warp past the end (never with kSub)
  const uint64_t e0 = (uint64_t)b * n + w0, e1 = (uint64_t)b * n + w1;
  uint64_t a0 = e0;  // smem index 0 holds element a0
  if ((((uintptr_t)s | (uintptr_t)t) & 15u) == 0) {
    a0 = e0 & ~uint64_t(3);
    const uint64_t v1 = e1 & ~uint64_t(3);  // [a0, v1) by float4, [v1, e1) scalar
    const int nv = (int)((v1 - a0) >> 2);  // <= (32 * kLeaf + 3) / 4 + 1 = 129
    // every load of the warp's range issued before any is stored (the
    // range is at most 5 float4 per lane and array)
    constexpr int kPer = (32 * kLeaf / 4 + 2 + 31) / 32;
    float4 va[kPer], vb[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
        va[j] = __ldg(reinterpret_cast<const float4*>(s + a0) + i);
        vb[j] = __ldg(reinterpret_cast<const float4*>(t + a0) + i);
      }
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int i = lane + 32 * j;
      if (i < nv) {
        reinterpret_cast<float4*>(ss[warp][0])[i] = va[j];
        reinterpret_cast<float4*>(ss[warp][1])[i] = vb[j];
      }
    }
    const int tail = (int)(e1 - v1);
    if (lane < tail) {
      ss[warp][0][(v1 - a0) + lane] = __ldg(s + v1 + lane);
      ss[warp][1][(v1 - a0) + lane] = __ldg(t + v1 + lane);
    }
  } else {
    const int cnt = (int)(e1 - e0);
    for (int i = lane; i < cnt; i += 32) {
      ss[warp][0][i] = __ldg(s + e0 + i);
      ss[warp][1][i] = __ldg(t + e0 + i);
    }
  }
  __syncwarp();
  double r = 0.0;
  if (g < groups) {
    const float* a = ss[warp][0] + ((uint64_t)b * n + lo - a0);
    const float* c = ss[warp][1] + ((uint64_t)b * n + lo - a0);
    auto fold = [&](int k0, int k1) {
      double acc = 0.0;
      for (int k = k0; k < k1; ++k) acc = __dadd_rn(acc, mse_term(a[k], c[k]));
      return acc;
    };
    if (m <= 8) {
      r = fold(0, (int)m);
    } else {
      const int h = (int)(m >> 1);
      r = __dadd_rn(fold(0, h), fold(h, (int)m));
    }
  }
  if constexpr (!kSub) {
    if (g < groups) out[((uint64_t)b << depth) + g] = r;
  } else {
    for (int o = 1; o < 32; o <<= 1) r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (lane == 0) wsum[warp] = r;
    __syncthreads();
    if (threadIdx.x == 0) {
      const double v = __dadd_rn(__dadd_rn(__dadd_rn(wsum[0], wsum[1]), __dadd_rn(wsum[2], wsum[3])),
                                 __dadd_rn(__dadd_rn(wsum[4], wsum[5]), __dadd_rn(wsum[6], wsum[7])));
      out[((uint64_t)b << (depth - kMseSubLog)) + blockIdx.x] = v;
    }
  }
}

// Perfect-tree halving: per pair y = blockIdx.y (cnt values each), CTA x
// reduces in[2048 x .. 2048 x + 2048) (a power of two count `cnt` <= 2048
// when fewer remain) to out[x]. On the last pass the single result per pair
// is divided by `div` into res[y * res_stride].
__global__ void __launch_bounds__(kRedThreads) halve_kernel(const double* in, uint32_t cnt,
                                                            double* out, double div, double* res,
                                                            uint32_t res_stride) {
  __shared__ double sm[2 * kRedThreads];
  const uint32_t per = cnt < 2u * kRedThreads ? cnt : 2u * kRedThreads;
  in += (uint64_t)blockIdx.y * cnt;
  out += (uint64_t)blockIdx.y * (cnt / per);
  const uint64_t base = (uint64_t)blockIdx.x * per;
  for (uint32_t i = threadIdx.x; i < per; i += kRedThreads) sm[i] = in[base + i];
  __syncthreads();
  for (uint32_t w = per >> 1; w >= 1; w >>= 1) {
    double v = 0.0;
    if (threadIdx.x < w) v = __dadd_rn(sm[2 * threadIdx.x], sm[2 * threadIdx.x + 1]);
    __syncthreads();
    if (threadIdx.x < w) sm[threadIdx.x] = v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (res) res[(uint64_t)blockIdx.y * res_stride] = __ddiv_rn(sm[0], div);
    else out[blockIdx.x] = sm[0];
  }
}

// pairwise_sum(terms of pair b, n) / div -> res[b * res_stride] for the nb
// pairs, via scratch `ws` (>= nb * (2^D + 2^D/2048) doubles).
// Halving passes over nb x 2^depth leaf sums already in ws.
cudaError_t halve_all(uint32_t depth, uint32_t nb, double div, double* res, uint32_t res_stride, double* ws,
                      cudaStream_t st, int* launches);

template <typename Term>
cudaError_t pairwise_sum_dev(const Term& f, uint64_t n, uint32_t nb, double div, double* res,
                             uint32_t res_stride, double* ws, cudaStream_t st, int* launches) {
  const uint32_t depth = tree_depth(n);
  const uint32_t groups = 1u << depth;
  leaf_sums_kernel<Term><<<dim3((groups + 255) / 256, nb), 256, 0, st>>>(f, n, depth, ws);
  ++*launches;
  return halve_all(depth, nb, div, res, res_stride, ws, st, launches);
}

cudaError_t halve_all(uint32_t depth, uint32_t nb, double div, double* res, uint32_t res_stride, double* ws,
                      cudaStream_t st, int* launches) {
  const uint32_t groups = 1u << depth;
  double* in = ws;
  double* out = ws + (uint64_t)nb * groups;
  uint32_t cnt = groups;
  for (;;) {
    const uint32_t per = cnt < 2u * kRedThreads ? cnt : 2u * kRedThreads;
    const uint32_t blocks = cnt / per;
    halve_kernel<<<dim3(blocks, nb), kRedThreads, 0, st>>>(in, cnt, out, div, blocks == 1 ? res : nullptr,
                                                          res_stride);
    ++*launches;
    if (blocks == 1) break;
    double* t = in;
    in = out;
    out = t;
    cnt = blocks;
  }
  return cudaGetLastError();
}

// Per-location cosine + its gradient (distill.hpp:94-121), then the
// trainer's chunk scaling of the whole gradient column (distill.hpp:245).
// One thread per (pair, location): the channel loops are sequential in the
// reference order; the loads of a channel step are independent of the
// accumulations, so unrolling keeps several in flight.
__global__ void __launch_bounds__(256, 4) cosine_kernel(const float* __restrict__ s, const float* __restrict__ t,
                              float* __restrict__ ds, uint64_t c, uint64_t hw, double w,
                              double gscale, double n, double* __restrict__ cos_loc) {
  const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= hw) return;
  const uint64_t pair = blockIdx.y;
  s += pair * c * hw;
  t += pair * c * hw;
  ds += pair * c * hw;
  cos_loc += pair * hw;
  double dot = 0.0, na2 = 0.0, nb2 = 0.0;
#pragma unroll 16
  for (uint64_t ch = 0; ch < c; ++ch) {
    const double a = (double)__ldg(s + ch * hw + p);
    const double b = (double)__ldg(t + ch * hw + p);
    dot = __dadd_rn(dot, __dmul_rn(a, b));
    na2 = __dadd_rn(na2, __dmul_rn(a, a));
    nb2 = __dadd_rn(nb2, __dmul_rn(b, b));
  }
  const bool zero = na2 == 0.0 || nb2 == 0.0;  // guarded: cos 0, no gradient
  double cosv = 0.0, nrm = 1.0;
  if (!zero) {
    nrm = __dsqrt_rn(__dmul_rn(na2, nb2));
    cosv = __ddiv_rn(dot, nrm);
  }
  // the per-element divisions by n, nrm and na2 use hoisted reciprocals and
  // two Markstein corrections (correctly rounded, qfb_device.cuh
  // markstein2_div; a zero numerator may come out +0 instead of -0, which
  // the following float additions to a non-negative-zero g cannot observe)
  DivCtx dn, dr, da;
  dn.s = n;
  dn.y = __drcp_rn(n);
  dr.s = nrm;
  dr.y = __drcp_rn(nrm);
  da.s = zero ? 1.0 : na2;
  da.y = __drcp_rn(da.s);
  cos_loc[p] = cosv;
#pragma unroll 8
  for (uint64_t ch = 0; ch < c; ++ch) {
    const uint64_t i = ch * hw + p;
    const double a = (double)__ldg(s + i);
    const double b = (double)__ldg(t + i);
    // MSE part (distill.hpp:89-90): 0.0f + float(2d/n)
    float g = __fadd_rn(0.0f, __double2float_rn(markstein2_div(__dmul_rn(2.0, __dadd_rn(a, -b)), dn)));
    if (!zero) {
      const double q = __dadd_rn(markstein2_div(b, dr), -markstein2_div(__dmul_rn(cosv, a), da));
      g = __fadd_rn(g, __double2float_rn(__dmul_rn(-w, q)));
    }
    ds[i] = __double2float_rn(__dmul_rn((double)g, gscale));
  }
}

// Adam (distill.hpp:264-279); the update is skipped when any gradient is
// non-finite (all_finite, distill.hpp:254-258): flag[0] counts them.
__global__ void nonfinite_kernel(const double* __restrict__ g, int64_t n, uint32_t* flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(g[i])) atomicAdd(flag, 1u);
}

__global__ void adam_kernel(double* __restrict__ p, double* __restrict__ m, double* __restrict__ v,
                            const double* __restrict__ g, int64_t n, double b1, double b2, double lr,
                            double eps, double bc1, double bc2, const uint32_t* flag) {
  if (*flag != 0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    const double mk = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dadd_rn(1.0, -b1), gi));
    const double vk = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dadd_rn(1.0, -b2), gi), gi));
    m[i] = mk;
    v[i] = vk;
    const double mhat = __ddiv_rn(mk, bc1);
    const double vhat = __ddiv_rn(vk, bc2);
    p[i] = __dadd_rn(p[i], -__ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
  }
}

// Device-stepped Adam for CUDA-graph replays: t = (non-skipped steps so
// far) + 1 read from counters[0] (distill.hpp:262-264: t = step - skipped),
// the bias corrections taken from a host-computed table (the host libm pow,
// bit-identical to the reference's), the skip decided from the gradient and
// loss non-finite counts in flag[0]. counters[1] counts skipped steps; a
// step beyond the table is skipped and latched in counters[2].
__global__ void nonfinite2_kernel(const double* __restrict__ g, int64_t n, const double* __restrict__ loss,
                                  int64_t n_loss, uint32_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n + n_loss; i += stride) {
    const double v = i < n ? g[i] : loss[i - n];
    if (!isfinite(v)) atomicAdd(flag, 1u);
  }
}

__global__ void adam_dev_kernel(double* __restrict__ p, double* __restrict__ m, double* __restrict__ v,
                                const double* __restrict__ g, int64_t n, double b1, double b2, double lr,
                                double eps, const double* __restrict__ bc, int64_t t_max,
                                const int64_t* __restrict__ counters, const uint32_t* flag) {
  const int64_t t = counters[0] + 1;
  if (*flag != 0 || t > t_max) return;
  const double bc1 = bc[2 * (t - 1)], bc2 = bc[2 * (t - 1) + 1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    const double mk = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dadd_rn(1.0, -b1), gi));
    const double vk = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dadd_rn(1.0, -b2), gi), gi));
    m[i] = mk;
    v[i] = vk;
    const double mhat = __ddiv_rn(mk, bc1);
    const double vhat = __ddiv_rn(vk, bc2);
    p[i] = __dadd_rn(p[i], -__ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
  }
}

__global__ void adam_advance_kernel(int64_t* counters, int64_t t_max, const uint32_t* flag) {
  const bool over = counters[0] + 1 > t_max;
  if (*flag != 0 || over) {
    counters[1] += 1;
    if (over) counters[2] = 1;
  } else {
    counters[0] += 1;
  }
}

// Row-order fold of per-frame gradient rows (the multi-GPU exchange's
// combine step): out[j] = ((into[j] + r0[j]) + r1[j]) + ..., one thread per
// column, so the bits equal the single-process frame-order accumulation.
__global__ void fold_rows_kernel(const double* __restrict__ rows, int64_t nrows, int64_t n,
                                 const double* __restrict__ into, double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = into ? __dadd_rn(into[j], rows[j]) : rows[j];
  for (int64_t r = 1; r < nrows; ++r) acc = __dadd_rn(acc, rows[r * n + j]);
  out[j] = acc;
}

}  // namespace
}  // namespace qfb

using namespace qfb;

namespace {

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~Guard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

qfb_status err(qfb_status st, const std::string& m) { return set_error(st, m.c_str()); }

}  // namespace

extern "C" {

qfb_status qfb_distill_batch(qfb_ctx* ctx, const float* student, const float* teacher, int64_t pairs,
                             int64_t channels, int64_t hw, double lambda_cos, double grad_scale,
                             float* d_student, double* out) {
  if (!ctx) return err(QFB_ERR_VALUE, "null qfb_ctx");
  if (channels < 1) return err(QFB_ERR_SHAPE, "distill_loss: channel dim must be >= 1");
  if (hw < 1 || pairs < 1) return err(QFB_ERR_SHAPE, "distill_loss: non-positive size");
  if (pairs > 65535) return err(QFB_ERR_UNSUPPORTED, "distill_batch: at most 65535 pairs per call");
  if (!student || !teacher || !d_student || !out) return err(QFB_ERR_VALUE, "distill_pair: null pointer");
  Guard g(ctx_device(ctx));
  const cudaStream_t st = ctx_stream(ctx);
  const uint64_t n = (uint64_t)channels * (uint64_t)hw;
  const uint32_t nb = (uint32_t)pairs;
  const uint64_t groups_n = 1ull << tree_depth(n), groups_hw = 1ull << tree_depth((uint64_t)hw);
  if (groups_n >= (1ull << 31)) return err(QFB_ERR_UNSUPPORTED, "distill_pair: tensor too large");
  void *ws = nullptr, *cl = nullptr;
  const uint64_t gmax = groups_n > groups_hw ? groups_n : groups_hw;
  if (qfb_status s = ctx_scratch(ctx, 0, nb * (gmax + gmax / 2048 + 2) * sizeof(double), &ws)) return s;
  if (qfb_status s = ctx_scratch(ctx, 1, nb * (uint64_t)hw * sizeof(double), &cl)) return s;
  int launches = 0;
  // MSE (+ d_s = float(2d/n)) then per-location cosine (+ its gradient and
  // the chunk scaling), then the mean cosine over locations
  const uint32_t depth_n = tree_depth(n);
  const uint32_t per_cta = 32u * kMseWarps;
  const dim3 mse_grid(((1u << depth_n) + per_cta - 1) / per_cta, nb);
  const bool sub = depth_n >= (uint32_t)kMseSubLog;  // CTAs reduce whole subtrees
  if (sub)
    mse_leaf_kernel<true><<<mse_grid, per_cta, 0, st>>>(student, teacher, n, depth_n, static_cast<double*>(ws));
  else
    mse_leaf_kernel<false><<<mse_grid, per_cta, 0, st>>>(student, teacher, n, depth_n, static_cast<double*>(ws));
  ++launches;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess)
    e = halve_all(sub ? depth_n - kMseSubLog : depth_n, nb, (double)n, out, 2, static_cast<double*>(ws), st,
                  &launches);
  if (e == cudaSuccess) {
    const double w = lambda_cos / (double)hw;
    cosine_kernel<<<dim3((unsigned)(((uint64_t)hw + 255) / 256), nb), 256, 0, st>>>(
        student, teacher, d_student, (uint64_t)channels, (uint64_t)hw, w, grad_scale, (double)n,
        static_cast<double*>(cl));
    ++launches;
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = pairwise_sum_dev(LoadTerm{static_cast<const double*>(cl), (uint64_t)hw}, (uint64_t)hw, nb, (double)hw,
                         out + 1, 2, static_cast<double*>(ws), st, &launches);
  ctx_count_launches(ctx, launches);
  if (e != cudaSuccess) return cuda_error(e, "distill_batch");
  return QFB_OK;
}

qfb_status qfb_distill_pair(qfb_ctx* ctx, const float* student, const float* teacher,
                            int64_t channels, int64_t hw, double lambda_cos, double grad_scale,
                            float* d_student, double* out2) {
  return qfb_distill_batch(ctx, student, teacher, 1, channels, hw, lambda_cos, grad_scale, d_student, out2);
}

qfb_status qfb_distill_loss_host(qfb_ctx* ctx, const float* f_s, const float* f_t, int64_t f_channels,
                                 int64_t f_hw, const float* i_s, const float* i_t, int64_t i_channels,
                                 int64_t i_hw, double lambda_cos, double grad_scale, double* out5,
                                 float* d_features, float* d_descriptors) {
  if (!ctx) return err(QFB_ERR_VALUE, "null qfb_ctx");
  if (!f_s || !f_t || !i_s || !i_t || !out5 || !d_features || !d_descriptors)
    return err(QFB_ERR_VALUE, "distill_loss_host: null pointer");
  if (f_channels < 1 || i_channels < 1) return err(QFB_ERR_SHAPE, "distill_loss: channel dim must be >= 1");
  if (f_hw < 1 || i_hw < 1) return err(QFB_ERR_SHAPE, "distill_loss: non-positive spatial size");
  Guard g(ctx_device(ctx));
  const cudaStream_t st = ctx_stream(ctx);
  const size_t nf = (size_t)f_channels * (size_t)f_hw, ni = (size_t)i_channels * (size_t)i_hw;
  void* buf = nullptr;
  if (qfb_status s = ctx_scratch(ctx, 2, (3 * nf + 3 * ni) * sizeof(float) + 4 * sizeof(double), &buf)) return s;
  float* b = static_cast<float*>(buf);
  float *dfs = b, *dft = b + nf, *ddf = b + 2 * nf, *dis = b + 3 * nf, *dit = dis + ni, *ddi = dis + 2 * ni;
  double* dout = reinterpret_cast<double*>(dis + 3 * ni);
  cudaError_t e = cudaMemcpyAsync(dfs, f_s, nf * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dft, f_t, nf * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dis, i_s, ni * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dit, i_t, ni * 4, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_error(e, "distill_loss_host H2D");
  if (qfb_status s = qfb_distill_pair(ctx, dfs, dft, f_channels, f_hw, lambda_cos, grad_scale, ddf, dout)) return s;
  if (qfb_status s = qfb_distill_pair(ctx, dis, dit, i_channels, i_hw, lambda_cos, grad_scale, ddi, dout + 2)) return s;
  double h[4];
  e = cudaMemcpyAsync(h, dout, sizeof h, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_features, ddf, nf * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_descriptors, ddi, ni * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_error(e, "distill_loss_host D2H");
  // distill.hpp:136-139: total, in the reference's evaluation order
  out5[1] = h[0];
  out5[2] = h[2];
  out5[3] = h[1];
  out5[4] = h[3];
  out5[0] = h[0] + h[2] + lambda_cos * (1.0 - h[1]) + lambda_cos * (1.0 - h[3]);
  return QFB_OK;
}

qfb_status qfb_fold_rows(qfb_ctx* ctx, const double* rows, int64_t nrows, int64_t n, const double* into,
                         double* out) {
  if (!ctx) return err(QFB_ERR_VALUE, "null qfb_ctx");
  if (nrows < 1 || n < 0 || (n > 0 && (!rows || !out))) return err(QFB_ERR_VALUE, "fold_rows: bad arguments");
  if (n == 0) return QFB_OK;
  Guard g(ctx_device(ctx));
  fold_rows_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx_stream(ctx)>>>(rows, nrows, n, into, out);
  ctx_count_launches(ctx, 1);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? QFB_OK : cuda_error(e, "fold_rows");
}

qfb_status qfb_adam_bias_corrections(double beta1, double beta2, int64_t t, double* bc1, double* bc2) {
  if (!bc1 || !bc2) return err(QFB_ERR_VALUE, "adam_bias_corrections: null pointer");
  if (t < 1) return err(QFB_ERR_VALUE, "adam_bias_corrections: step must be >= 1");
  *bc1 = 1.0 - std::pow(beta1, (double)t);  // distill.hpp:265-266 (host libm pow)
  *bc2 = 1.0 - std::pow(beta2, (double)t);
  return QFB_OK;
}

qfb_status qfb_adam_step(qfb_ctx* ctx, double* params, double* m, double* v, const double* grads,
                         int64_t n, double beta1, double beta2, double lr, double eps, double bc1,
                         double bc2, uint32_t* skipped) {
  if (!ctx) return err(QFB_ERR_VALUE, "null qfb_ctx");
  if (n < 0 || (n > 0 && (!params || !m || !v || !grads)) || !skipped)
    return err(QFB_ERR_VALUE, "adam_step: bad arguments");
  Guard g(ctx_device(ctx));
  const cudaStream_t st = ctx_stream(ctx);
  cudaError_t e = cudaMemsetAsync(skipped, 0, sizeof(uint32_t), st);
  const int blocks = (int)((n + 255) / 256 > 1024 ? 1024 : (n + 255) / 256);
  if (e == cudaSuccess && n > 0) {
    nonfinite_kernel<<<blocks, 256, 0, st>>>(grads, n, skipped);
    adam_kernel<<<blocks, 256, 0, st>>>(params, m, v, grads, n, beta1, beta2, lr, eps, bc1, bc2, skipped);
    ctx_count_launches(ctx, 2);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return cuda_error(e, "adam_step");
  return QFB_OK;
}

qfb_status qfb_adam_bias_table(double beta1, double beta2, int64_t t_max, double* table) {
  if (!table || t_max < 1) return err(QFB_ERR_VALUE, "adam_bias_table: bad arguments");
  for (int64_t t = 1; t <= t_max; ++t)
    if (qfb_status s = qfb_adam_bias_corrections(beta1, beta2, t, table + 2 * (t - 1), table + 2 * (t - 1) + 1))
      return s;
  return QFB_OK;
}

qfb_status qfb_adam_step_dev(qfb_ctx* ctx, double* params, double* m, double* v, const double* grads,
                             int64_t n, double beta1, double beta2, double lr, double eps,
                             const double* bias_table, int64_t t_max, int64_t* counters,
                             const double* loss, int64_t n_loss, uint32_t* flag) {
  if (!ctx) return err(QFB_ERR_VALUE, "null qfb_ctx");
  if (n < 0 || (n > 0 && (!params || !m || !v || !grads)) || !flag || !counters || !bias_table ||
      t_max < 1 || n_loss < 0 || (n_loss > 0 && !loss))
    return err(QFB_ERR_VALUE, "adam_step_dev: bad arguments");
  Guard g(ctx_device(ctx));
  const cudaStream_t st = ctx_stream(ctx);
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(uint32_t), st);
  const int64_t work = n + n_loss;
  const int blocks = (int)((work + 255) / 256 > 1024 ? 1024 : ((work + 255) / 256 > 0 ? (work + 255) / 256 : 1));
  if (e == cudaSuccess) {
    nonfinite2_kernel<<<blocks, 256, 0, st>>>(grads, n, loss, n_loss, flag);
    adam_dev_kernel<<<blocks, 256, 0, st>>>(params, m, v, grads, n, beta1, beta2, lr, eps, bias_table, t_max,
                                            counters, flag);
    adam_advance_kernel<<<1, 1, 0, st>>>(counters, t_max, flag);
    ctx_count_launches(ctx, 3);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return cuda_error(e, "adam_step_dev");
  return QFB_OK;
}

}  // extern "C"
