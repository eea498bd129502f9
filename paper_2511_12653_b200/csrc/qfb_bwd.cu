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
// at depth D ("leaf groups", <= 16 elements each), and a group's own sum is
// fold(first half) + fold(second half) (or one fold if <= 8). Node
// boundaries follow the recursive floor split, located per group by
// descending the bits of its index. A perfect tree is exactly what an xor
// butterfly computes (IEEE addition is commutative), so:
//   tile    = 2^g consecutive leaf groups (g = min(D, 8)), <= 4096 elements:
//             16-byte vector window loads (coalesced) -> per-element term
//             (double) in padded smem, d_input straight to HBM -> one leaf
//             group per thread -> warp/CTA butterfly = the subtree's sum;
//   segment = one row: its 2^(D-g) tile partials are reduced in tree order
//             by the last CTA to finish (threadfence + atomic ticket);
//   channel = rows of the same channel over `outer` are accumulated in row
//             order by the last segment to finish (the trainer's `g += ...`).
// CTAs are persistent (grid = SMs x resident CTAs) and stride over tiles.
// The result is bit-identical to the reference for any grid size.
// tests/test_tree_model.py executes this exact schedule on the CPU.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "qfb_device.cuh"
#include "qfb_kernels.h"

namespace qfb {

namespace {

constexpr int kPadShift = 4;  // one pad double every 16: conflict-light leaf reads
constexpr int kSmemDoubles = kBwdTileMax + (kBwdTileMax >> kPadShift);

__device__ __forceinline__ int pad_idx(int e) { return e + (e >> kPadShift); }

// Descend `levels` levels of the reference split from node (lo, m) along
// the bits of `path` (MSB first): bit 0 = left child [lo, lo + m/2),
// bit 1 = right child [lo + m/2, lo + m).
template <typename I>
__device__ __forceinline__ void descend(I& lo, I& m, uint32_t path, int levels) {
  for (int l = levels - 1; l >= 0; --l) {
    const I h = m >> 1;
    if ((path >> l) & 1u) {
      lo += h;
      m -= h;
    } else {
      m = h;
    }
  }
}

// Left fold from 0.0 over smem[start, start + len), len <= 8
// (tensor.hpp:101-104), as a fixed-trip predicated loop.
__device__ __forceinline__ double fold8(const double* sm, int start, int len) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (k < len) acc = __dadd_rn(acc, sm[pad_idx(start + k)]);
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

// Per-element terms of one element (quant.hpp:217-228 + :250-251).
struct ElemOut {
  float dx;
  double term;
};

__device__ __forceinline__ ElemOut elem_terms(float xv, float uv, double s, double q) {
  const GradTerm gt = grad_term(xv, s, q);
  return {masked_upstream(gt.mask, uv), __dmul_rn(gt.d_ds, (double)uv)};
}

template <typename T>
struct VecIO;

template <>
struct VecIO<float> {
  static constexpr int V = 4;
  __device__ __forceinline__ static void unpack(const uint4& r, float* v) { Elem<float>::unpack(r, v); }
  __device__ __forceinline__ static uint4 pack(const float* v) {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
  }
  __device__ __forceinline__ static void store1(void* p, uint64_t i, float v) {
    static_cast<float*>(p)[i] = v;
  }
};

template <>
struct VecIO<__half> {
  static constexpr int V = 8;
  __device__ __forceinline__ static void unpack(const uint4& r, float* v) { Elem<__half>::unpack(r, v); }
  // dx values are +-up, +-0 or NaN of a half upstream: exact in binary16
  __device__ __forceinline__ static uint4 pack(const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      w[i] = (uint32_t)__half_as_ushort(__float2half_rn(v[2 * i])) |
             ((uint32_t)__half_as_ushort(__float2half_rn(v[2 * i + 1])) << 16);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ static void store1(void* p, uint64_t i, float v) {
    static_cast<__half*>(p)[i] = __float2half_rn(v);
  }
};

template <typename T>
__device__ __forceinline__ float load1(const void* p, uint64_t i) {
  if constexpr (sizeof(T) == 4) {
    return __ldg(static_cast<const float*>(p) + i);
  } else {
    return __half2float(static_cast<const __half*>(p)[i]);
  }
}

// Pass 1, vector window: units of V elements aligned to 16 bytes covering
// [A, A + m); elements outside the tile are loaded but ignored.
template <typename T>
__device__ __forceinline__ void pass1_vec(const BwdDesc& d, uint64_t A, int m, double s, double q,
                                          double* sm) {
  constexpr int V = VecIO<T>::V;
  const int off = (int)(A & (V - 1));
  const uint64_t ubase = A >> (V == 4 ? 2 : 3);
  const int U = (off + m + V - 1) / V;
  const uint4* xv = static_cast<const uint4*>(d.x) + ubase;
  const uint4* uv = static_cast<const uint4*>(d.up) + ubase;
  uint4* dxv = d.dx ? static_cast<uint4*>(d.dx) + ubase : nullptr;
  for (int u0 = threadIdx.x; u0 < U; u0 += 2 * kBwdThreads) {
    uint4 rx[2], ru[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int u = u0 + k * kBwdThreads;
      if (u < U) {
        rx[k] = ld_nc_v4(xv + u);
        ru[k] = ld_nc_v4(uv + u);
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int u = u0 + k * kBwdThreads;
      if (u >= U) break;
      float x[V], up[V], dx[V];
      VecIO<T>::unpack(rx[k], x);
      VecIO<T>::unpack(ru[k], up);
      const int e0 = u * V - off;  // tile-relative index of element 0
      const bool full = e0 >= 0 && e0 + V <= m;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const ElemOut eo = elem_terms(x[j], up[j], s, q);
        dx[j] = eo.dx;
        const int e = e0 + j;
        if (full || (unsigned)e < (unsigned)m) sm[pad_idx(e)] = eo.term;
      }
      if (dxv != nullptr) {
        if (full) {
          st_v4(dxv + u, VecIO<T>::pack(dx), false);
        } else {
#pragma unroll
          for (int j = 0; j < V; ++j)
            if ((unsigned)(e0 + j) < (unsigned)m) VecIO<T>::store1(d.dx, A + e0 + j, dx[j]);
        }
      }
    }
  }
}

// Pass 1, scalar (unaligned buffers).
template <typename T>
__device__ __forceinline__ void pass1_scalar(const BwdDesc& d, uint64_t A, int m, double s,
                                             double q, double* sm) {
  for (int e = threadIdx.x; e < m; e += kBwdThreads) {
    const ElemOut eo = elem_terms(load1<T>(d.x, A + e), load1<T>(d.up, A + e), s, q);
    if (d.dx != nullptr) VecIO<T>::store1(d.dx, A + e, eo.dx);
    sm[pad_idx(e)] = eo.term;
  }
}

template <typename T>
__global__ void __launch_bounds__(kBwdThreads, 4)
    bwd_kernel(const __grid_constant__ BwdBatch bt) {
  __shared__ double sm[kSmemDoubles];
  __shared__ double red[kBwdThreads / 32];
  __shared__ int last_flag;
  const int tid = threadIdx.x;
  const uint32_t total = bt.tile_begin[bt.n];

  for (uint32_t tile_id = blockIdx.x; tile_id < total; tile_id += gridDim.x) {
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

    // Tile root: node t at depth D - g of the row's tree (64-bit: rows may
    // exceed 2^32 elements); everything inside a tile fits 32 bits.
    uint64_t lo = 0, mm = d.inner;
    descend<uint64_t>(lo, mm, t, (int)d.tps_log);
    const int m = (int)mm;  // <= kBwdTileMax
    const uint64_t A = (uint64_t)seg * d.inner + lo;
    const double s = d.s64[c];
    const double q = d.q;

    if (d.vec) pass1_vec<T>(d, A, m, s, q, sm);
    else pass1_scalar<T>(d, A, m, s, q, sm);
    __syncthreads();

    // Pass 2: one leaf group per thread, then the perfect-tree butterfly.
    const int groups = 1 << d.g;
    double v = 0.0;
    if (tid < groups) {
      int glo = 0, gm = m;
      descend<int>(glo, gm, (uint32_t)tid, (int)d.g);
      const int h = gm > 8 ? gm >> 1 : gm;
      v = fold8(sm, glo, h);
      if (gm > 8) v = __dadd_rn(v, fold8(sm, glo + h, gm - h));
    }
    const double tile_sum = cta_tree_sum(v, groups, red);

    const uint32_t tps = 1u << d.tps_log;
    if (tps == 1) {
      if (tid == 0) finish_segment(d, seg, c, __dmul_rn(tile_sum, d.chain[c]));
    } else {
      // Pass 3: segment completion by the last tile (atomic ticket).
      if (tid == 0) {
        d.partials[(uint64_t)seg * tps + t] = tile_sum;
        __threadfence();
        const uint32_t ticket = atomicAdd(d.seg_counters + seg, 1u);
        last_flag = (ticket == tps - 1);
      }
      __syncthreads();
      if (last_flag) {
        __threadfence();
        const double* p = d.partials + (uint64_t)seg * tps;
        // Each thread reduces `per` consecutive partials as a perfect
        // subtree, then the CTA butterfly combines the subtrees in order.
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
              // per > 16 (rows > 2^26 elements): level-by-level in place
              // over the thread's own slice, still the perfect-tree order.
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
    }
    __syncthreads();  // smem / red / last_flag are reused by the next tile
  }
}

}  // namespace

cudaError_t bwd_occupancy(int dtype, int* blocks_per_sm) {
  const void* f = dtype == 0 ? (const void*)bwd_kernel<float> : (const void*)bwd_kernel<__half>;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, kBwdThreads, 0);
}

cudaError_t launch_bwd(int dtype, const BwdBatch& b, int grid, cudaStream_t st) {
  const uint32_t tiles = b.tile_begin[b.n];
  if (tiles == 0) return cudaSuccess;
  if ((uint32_t)grid > tiles) grid = (int)tiles;
  if (dtype == 0) bwd_kernel<float><<<grid, kBwdThreads, 0, st>>>(b);
  else bwd_kernel<__half><<<grid, kBwdThreads, 0, st>>>(b);
  return cudaGetLastError();
}

}  // namespace qfb
