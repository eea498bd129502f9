// qfb_bwd.cu — scale-only STE/LSQ backward with the reference's pairwise
// reduction tree reproduced exactly on the device.
//
// Reference: quant.hpp:217-294 (per-element terms in double, d_input =
// mask * upstream, d_log_s = pairwise_sum(terms) * chain) and
// tensor.hpp:100-109 (pairwise_sum: n <= 8 -> left fold from 0.0, else
// split h = n/2 and add the two halves).
//
// Tree decomposition. For a row of n elements let D be the smallest depth
// with ceil(n / 2^D) <= 16. Every node above depth D has > 16 > 8 elements,
// so the top of the reference tree is a PERFECT binary tree with 2^D nodes
// at depth D ("leaf groups", 9..16 or fewer elements each), and a group's
// own sum is fold(first half) + fold(second half) (or one fold if <= 8).
// Node boundaries follow the recursive floor split, computed per group by
// descending the bits of its index. A perfect tree is exactly what an xor
// butterfly computes (IEEE addition is commutative), so:
//   tile   = 2^g consecutive leaf groups (g = min(D, 8)), one CTA;
//            elementwise pass (coalesced) -> per-element term in smem ->
//            one leaf group per thread -> warp/CTA butterfly = subtree sum;
//   segment (one row): 2^(D-g) tile partials, reduced in tree order by the
//            last CTA to finish (threadfence + atomic ticket, no extra launch);
//   channel: rows of the same channel over `outer` are accumulated in row
//            order by the last segment to finish (the trainer's `g += ...`).
// The result is bit-identical to the reference for any grid size.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "qfb_device.cuh"
#include "qfb_kernels.h"

namespace qfb {

namespace {

constexpr int kPadShift = 4;  // one pad double every 16: conflict-free leaf reads
constexpr int kSmemDoubles = kBwdTileMax + (kBwdTileMax >> kPadShift);
constexpr int kElemsPerThread = kBwdTileMax / kBwdThreads;  // 16

__device__ __forceinline__ int pad_idx(int e) { return e + (e >> kPadShift); }

// Descend `levels` levels of the reference split from node (lo, m) along
// the bits of `path` (MSB first): bit 0 = left child [lo, lo + m/2),
// bit 1 = right child [lo + m/2, lo + m).
__device__ __forceinline__ void descend(uint64_t& lo, uint64_t& m, uint32_t path, int levels) {
  for (int l = levels - 1; l >= 0; --l) {
    const uint64_t h = m >> 1;
    if ((path >> l) & 1u) {
      lo += h;
      m -= h;
    } else {
      m = h;
    }
  }
}

// Left fold from 0.0 over smem[start, start + len), tensor.hpp:101-104.
__device__ __forceinline__ double fold(const double* sm, int start, int len) {
  double acc = 0.0;
  for (int k = 0; k < len; ++k) acc = __dadd_rn(acc, sm[pad_idx(start + k)]);
  return acc;
}

// Butterfly over the first `lanes` (power of two) threads of the CTA; the
// result (sum in perfect-tree order) is returned to thread 0.
__device__ __forceinline__ double cta_tree_sum(double v, int lanes, double* red) {
  const int tid = threadIdx.x;
  const int wl = lanes < 32 ? lanes : 32;
  for (int off = 1; off < wl; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  if (lanes <= 32) return v;
  const int nw = lanes >> 5;
  __syncthreads();
  if ((tid & 31) == 0 && (tid >> 5) < nw) red[tid >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (tid < 32) {
    r = tid < nw ? red[tid] : 0.0;
    for (int off = 1; off < nw; off <<= 1) r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, off));
  }
  return r;
}

// Perfect-tree sum of P consecutive partials (L2 loads: written by other CTAs).
template <int P>
__device__ __forceinline__ double tree_load(const double* p) {
  if constexpr (P == 1) {
    return __ldcg(p);
  } else {
    return __dadd_rn(tree_load<P / 2>(p), tree_load<P / 2>(p + P / 2));
  }
}

template <typename T>
__device__ __forceinline__ float load_elem(const void* p, uint64_t i) {
  if constexpr (sizeof(T) == 4) {
    return __ldg(static_cast<const float*>(p) + i);
  } else {
    return __half2float(static_cast<const __half*>(p)[i]);
  }
}

template <typename T>
__device__ __forceinline__ void store_elem(void* p, uint64_t i, float v) {
  if constexpr (sizeof(T) == 4) {
    static_cast<float*>(p)[i] = v;
  } else {
    static_cast<__half*>(p)[i] = __float2half_rn(v);  // v is +-up or +-0/NaN: exact
  }
}

// Channel-level completion: fold the per-row results of channel c in row
// order (frontend.hpp:222-228 accumulation).
__device__ void finish_segment(const BwdDesc& d, uint32_t seg, uint32_t c, double r) {
  if (d.outer == 1) {
    d.d_log_s[c] = d.accumulate ? __dadd_rn(d.d_log_s[c], r) : r;
    return;
  }
  d.seg_results[seg] = r;
  __threadfence();
  const uint32_t ticket = atomicAdd(d.chan_counters + c, 1u);
  if (ticket != d.outer - 1) return;
  __threadfence();
  double acc = d.accumulate ? __dadd_rn(d.d_log_s[c], __ldcg(d.seg_results + c))
                            : __ldcg(d.seg_results + c);
  for (uint32_t o = 1; o < d.outer; ++o)
    acc = __dadd_rn(acc, __ldcg(d.seg_results + (uint64_t)o * d.chans + c));
  d.d_log_s[c] = acc;
  d.chan_counters[c] = 0;  // self-reset for the next launch
}

template <typename T>
__global__ void __launch_bounds__(kBwdThreads, 4)
    bwd_kernel(const __grid_constant__ BwdBatch bt) {
  __shared__ double sm[kSmemDoubles];
  __shared__ double red[kBwdThreads / 32];
  __shared__ int last_flag;

  const uint32_t tile_id = blockIdx.x;
  int di = 0, hi = bt.n - 1;
  while (di < hi) {
    const int mid = (di + hi + 1) >> 1;
    if (bt.tile_begin[mid] <= tile_id) di = mid;
    else hi = mid - 1;
  }
  const BwdDesc& d = bt.d[di];
  const uint32_t local = tile_id - bt.tile_begin[di];
  const uint32_t seg = local >> d.tps_log;
  const uint32_t t = local & ((1u << d.tps_log) - 1u);
  const uint32_t c = seg % d.chans;
  const uint64_t row = (uint64_t)seg * d.inner;

  // Tile root: depth D - g node number t of the row's tree.
  uint64_t lo = 0, m = d.inner;
  descend(lo, m, t, (int)d.tps_log);
  const int tm = (int)m;  // <= kBwdTileMax
  const double s = d.s64[c];
  const double q = d.q;
  const int tid = threadIdx.x;

  // Pass 1: elementwise terms (coalesced), dx written straight to HBM.
  float xr[kElemsPerThread], ur[kElemsPerThread];
#pragma unroll
  for (int k = 0; k < kElemsPerThread; ++k) {
    const int e = tid + k * kBwdThreads;
    if (e < tm) {
      xr[k] = load_elem<T>(d.x, row + lo + e);
      ur[k] = load_elem<T>(d.up, row + lo + e);
    }
  }
#pragma unroll
  for (int k = 0; k < kElemsPerThread; ++k) {
    const int e = tid + k * kBwdThreads;
    if (e < tm) {
      const GradTerm gt = grad_term(xr[k], s, q);
      // d_input = float(mask * double(up)): +-up, or 0*up (+-0 / NaN)
      if (d.dx != nullptr) store_elem<T>(d.dx, row + lo + e, gt.mask ? ur[k] : __fmul_rn(0.0f, ur[k]));
      sm[pad_idx(e)] = __dmul_rn(gt.d_ds, (double)ur[k]);
    }
  }
  __syncthreads();

  // Pass 2: one leaf group per thread, then the perfect-tree butterfly.
  const int groups = 1 << d.g;
  double v = 0.0;
  if (tid < groups) {
    uint64_t glo = lo, gm = m;
    descend(glo, gm, (uint32_t)tid, (int)d.g);
    const int start = (int)(glo - lo);
    const int len = (int)gm;
    if (len <= 8) {
      v = fold(sm, start, len);
    } else {
      const int h = len >> 1;
      v = __dadd_rn(fold(sm, start, h), fold(sm, start + h, len - h));
    }
  }
  const double tile_sum = cta_tree_sum(v, groups, red);

  const uint32_t tps = 1u << d.tps_log;
  if (tps == 1) {
    if (tid == 0) finish_segment(d, seg, c, __dmul_rn(tile_sum, d.chain[c]));
    return;
  }

  // Pass 3: segment completion by the last tile (atomic ticket).
  if (tid == 0) {
    d.partials[(uint64_t)seg * tps + t] = tile_sum;
    __threadfence();
    const uint32_t ticket = atomicAdd(d.seg_counters + seg, 1u);
    last_flag = (ticket == tps - 1);
  }
  __syncthreads();
  if (!last_flag) return;
  __threadfence();
  const double* p = d.partials + (uint64_t)seg * tps;
  // Each thread reduces `per` consecutive partials as a perfect subtree,
  // then the CTA butterfly combines the 2^k subtrees in order.
  const uint32_t lanes = tps < (uint32_t)kBwdThreads ? tps : (uint32_t)kBwdThreads;
  const uint32_t per = tps / lanes;
  double w = 0.0;
  if ((uint32_t)tid < lanes) {
    const double* mine = p + (uint64_t)tid * per;
    switch (per) {
      case 1: w = tree_load<1>(mine); break;
      case 2: w = tree_load<2>(mine); break;
      case 4: w = tree_load<4>(mine); break;
      case 8: w = tree_load<8>(mine); break;
      case 16: w = tree_load<16>(mine); break;
      default: {
        // per > 16 (rows > 2^26 elements): level-by-level in place over the
        // thread's own slice, still the perfect-tree order.
        double* q2 = const_cast<double*>(mine);
        for (uint32_t width = per; width > 1; width >>= 1)
          for (uint32_t k = 0; k < width / 2; ++k)
            q2[k] = __dadd_rn(__ldcg(q2 + 2 * k), __ldcg(q2 + 2 * k + 1));
        w = __ldcg(q2);
      }
    }
  }
  const double seg_sum = cta_tree_sum(w, (int)lanes, red);
  if (tid == 0) {
    d.seg_counters[seg] = 0;  // self-reset
    finish_segment(d, seg, c, __dmul_rn(seg_sum, d.chain[c]));
  }
}

}  // namespace

cudaError_t launch_bwd(int dtype, const BwdBatch& b, cudaStream_t st) {
  const uint32_t tiles = b.tile_begin[b.n];
  if (tiles == 0) return cudaSuccess;
  if (dtype == 0) bwd_kernel<float><<<tiles, kBwdThreads, 0, st>>>(b);
  else bwd_kernel<__half><<<tiles, kBwdThreads, 0, st>>>(b);
  return cudaGetLastError();
}

}  // namespace qfb
