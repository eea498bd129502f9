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
//   tile    = 2^g consecutive leaf groups (g = min(D, 8)), <= 4096 elements,
//             staged into shared memory by the TMA engine (cp.async.bulk +
//             mbarrier, double-buffered: tile i+1 lands while tile i
//             computes); each thread owns one leaf group, computes its
//             elements' terms in registers and folds them in reference order,
//             writing d_input back into the stage; a coalesced 16-byte copy
//             moves d_input to HBM; warp/CTA butterfly = the subtree's sum;
//   segment = one row: its 2^(D-g) tile partials are reduced in tree order
//             by a small stream-ordered finisher kernel (one warp per
//             channel: per-lane perfect subtrees + xor butterfly), which also
//             applies the chain factor and folds the rows of a channel over
//             `outer` in row order (the trainer's `g += ...`). No fences,
//             atomics or tickets on the hot path.
// CTAs are persistent (grid = SMs x resident CTAs) and stride over tiles.
// The result is bit-identical to the reference for any grid size.
// tests/test_tree_model.py executes this exact schedule on the CPU.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "qfb_device.cuh"
#include "qfb_kernels.h"

namespace qfb {

namespace {

constexpr int kStages = 2;
constexpr int kWinPad = 32;  // window slack: 16-byte rounding at both ends

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

template <typename T>
struct Stage {
  T x[kBwdTileMax + kWinPad];
  T up[kBwdTileMax + kWinPad];
};

template <typename T>
__device__ __forceinline__ float to_f(T v) {
  if constexpr (sizeof(T) == 4) return v;
  else return __half2float(v);
}
template <typename T>
__device__ __forceinline__ T from_f(float v) {
  if constexpr (sizeof(T) == 4) return v;
  else return __float2half_rn(v);  // d_input of a half upstream: exact
}

// Where one tile lives: descriptor, row segment, tree node, its 16-byte
// window and the division context — computed once by the producer thread.
struct TileRef {
  int di;
  uint32_t seg, t, c;
  uint64_t A;   // first element (descriptor-relative)
  int m;        // elements
  int off;      // tile start inside the staged window (elements)
  uint64_t w0;  // window [w0, w1) in bytes
  uint64_t w1;
  double s, y;  // scale and RN(1/s)
};

__device__ __forceinline__ TileRef locate(const BwdBatch& bt, uint32_t tile_id) {
  TileRef r;
  int hi = bt.n - 1;
  r.di = 0;
  while (r.di < hi) {
    const int mid = (r.di + hi + 1) >> 1;
    if (bt.tile_begin[mid] <= tile_id) r.di = mid;
    else hi = mid - 1;
  }
  const BwdDesc& d = bt.d[r.di];
  const uint32_t local = tile_id - bt.tile_begin[r.di];
  r.seg = local >> d.tps_log;
  r.t = local & ((1u << d.tps_log) - 1u);
  r.c = r.seg % d.chans;
  // tile root: node t at depth D - g of the row's tree (64-bit: rows may
  // exceed 2^32 elements); everything inside a tile fits 32 bits
  uint64_t lo = 0, mm = d.inner;
  descend<uint64_t>(lo, mm, r.t, (int)d.tps_log);
  r.A = (uint64_t)r.seg * d.inner + lo;
  r.m = (int)mm;
  return r;
}

template <typename T>
__device__ __forceinline__ void window(const BwdDesc& d, const TileRef& r, uint64_t& w0,
                                       uint64_t& w1);

// Producer-side completion of a TileRef: window, in-stage offset, s, 1/s.
template <typename T>
__device__ __forceinline__ TileRef locate_full(const BwdBatch& bt, uint32_t tile_id) {
  TileRef r = locate(bt, tile_id);
  const BwdDesc& d = bt.d[r.di];
  window<T>(d, r, r.w0, r.w1);
  r.off = (int)((r.A * sizeof(T) - r.w0) / sizeof(T));
  r.s = d.s64[r.c];
  r.y = __drcp_rn(r.s);
  return r;
}

// 16-byte window [w0, w1) (bytes) of a tile that a bulk copy may fetch:
// never past the last full 16 bytes of the tensor (the few elements beyond
// are loaded by threads).
template <typename T>
__device__ __forceinline__ void window(const BwdDesc& d, const TileRef& r, uint64_t& w0,
                                       uint64_t& w1) {
  const uint64_t b0 = r.A * sizeof(T), b1 = (r.A + (uint64_t)r.m) * sizeof(T);
  const uint64_t tot = d.total_bytes;
  w0 = b0 & ~uint64_t(15);
  w1 = (b1 + 15) & ~uint64_t(15);
  const uint64_t cap = tot & ~uint64_t(15);
  if (w1 > cap) w1 = cap > w0 ? cap : w0;
}

// Thread 0: arm the stage's mbarrier and launch the two bulk copies.
template <typename T>
__device__ __forceinline__ void issue_tile(const BwdDesc& d, const TileRef& r, Stage<T>& st,
                                           uint64_t* bar) {
  const uint32_t bytes = (uint32_t)(r.w1 - r.w0);
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(bar, 2 * bytes);
  if (bytes) {
    bulk_g2s(st.x, static_cast<const char*>(d.x) + r.w0, bytes, bar);
    bulk_g2s(st.up, static_cast<const char*>(d.up) + r.w0, bytes, bar);
  }
}

// Group (leaf) of this thread inside a tile of m elements: depends only on
// (m, g), and a descriptor's tiles take at most two sizes -> 2-slot cache.
struct GroupCache {
  int k0 = -1, lo0 = 0, len0 = 0;
  int k1 = -1, lo1 = 0, len1 = 0;

  __device__ __forceinline__ void get(int m, int g, int tid, int& glo, int& glen) {
    const int k = m | (g << 16);
    if (k0 == k) {
      glo = lo0;
      glen = len0;
      return;
    }
    if (k1 == k) {
      glo = lo1;
      glen = len1;
      return;
    }
    int l = 0, mm = m;
    if (tid < (1 << g)) descend<int>(l, mm, (uint32_t)tid, g);
    else mm = 0;
    k1 = k0;
    lo1 = lo0;
    len1 = len0;
    k0 = k;
    lo0 = l;
    len0 = mm;
    glo = l;
    glen = mm;
  }
};

// Terms of one element: d_ds * up (double) and d_input (x86 NaN rules).
// Exact reference semantics for the rare elements the fast path cannot
// certify (zeros, inf/NaN, ties, binade edges): IEEE division, quant.hpp
// :217-228 verbatim. Out of line so it never bloats the hot loop.
static __device__ __noinline__ double2 slow_elem(float xv, float uv, double s, double q) {
  const GradTerm gt = grad_term(xv, s, q);
  return make_double2(__dmul_rn(gt.d_ds, (double)uv), (double)masked_upstream(gt.mask, uv));
}

// Pin a uniform double in a register (stops the compiler from
// rematerializing it from the dynamically indexed parameter bank per use).
__device__ __forceinline__ double pin(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}

// One element: term = d_ds * up (double) and d_input, with z = RN(x/s)
// from certified_quotient (qfb_device.cuh); uncertified elements take the
// exact IEEE path in slow_elem (returned in registers, never via memory).
template <typename T, bool kDx>
__device__ __forceinline__ double elem(T* sx, const T* su, int k, const DivCtx& dc, double q) {
  const float xv = to_f<T>(sx[k]);
  const float uv = to_f<T>(su[k]);
  double z;
  // one rare-path test: uncertified quotient or a non-finite upstream
  const bool up_finite = (__float_as_uint(uv) & 0x7f800000u) != 0x7f800000u;
  const bool ok = certified_quotient((double)xv, dc, z) && up_finite;
  const bool mask = fabs(z) <= q;
  const double d_ds = mask ? __dadd_rn(rint(z), -z) : copysign(q, z);
  double term = __dmul_rn(d_ds, (double)uv);
  float dx = mask ? uv : __uint_as_float(__float_as_uint(uv) & 0x80000000u);  // finite up
  if (__builtin_expect(!ok, 0)) {
    const double2 r = slow_elem(xv, uv, dc.s, q);
    term = r.x;
    dx = (float)r.y;  // exact: r.y is a float widened
  }
  if (kDx) sx[k] = from_f<T>(dx);
  return term;
}

// A leaf group's sum in the reference order: fold(left half) + fold(right
// half) from 0.0 each (or one fold if <= 8 elements). The two folds are
// independent chains, so they are interleaved for ILP.
template <typename T, bool kDx>
__device__ __forceinline__ double group_sum(T* sx, const T* su, int glen, const DivCtx& dc,
                                            double q) {
  if (glen <= 8) {
    double acc = 0.0;
    for (int k = 0; k < glen; ++k) acc = __dadd_rn(acc, elem<T, kDx>(sx, su, k, dc, q));
    return acc;
  }
  const int h = glen >> 1;  // left; right has glen - h >= h elements
  T* rx = sx + h;
  const T* ru = su + h;
  double acc_l = 0.0, acc_r = 0.0;
  for (int k = 0; k < h; ++k) {
    const double tl = elem<T, kDx>(sx, su, k, dc, q);
    const double tr = elem<T, kDx>(rx, ru, k, dc, q);
    acc_l = __dadd_rn(acc_l, tl);
    acc_r = __dadd_rn(acc_r, tr);
  }
  if (glen - h > h) acc_r = __dadd_rn(acc_r, elem<T, kDx>(rx, ru, h, dc, q));
  return __dadd_rn(acc_l, acc_r);
}

template <typename T>
__global__ void __launch_bounds__(kBwdThreads, 3) bwd_kernel(const __grid_constant__ BwdBatch bt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Stage<T>* stages = reinterpret_cast<Stage<T>*>(smem_raw);
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ TileRef sh_tile[2];
  __shared__ double red[kBwdThreads / 32];
  const int tid = threadIdx.x;
  const uint32_t total = bt.tile_begin[bt.n];
  if (blockIdx.x >= total) return;

  // Thread 0 is the producer: it locates tiles and issues their bulk copies
  // one tile ahead; everyone reads the tile descriptors from smem.
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    sh_tile[0] = locate_full<T>(bt, blockIdx.x);
    if (bt.d[sh_tile[0].di].vec) issue_tile<T>(bt.d[sh_tile[0].di], sh_tile[0], stages[0], &bars[0]);
  }
  __syncthreads();

  uint32_t phase_bits = 0;  // per-stage mbarrier parity
  GroupCache gc;
  int it = 0;
  for (uint32_t tile_id = blockIdx.x; tile_id < total; tile_id += gridDim.x, ++it) {
    const int sidx = it & (kStages - 1);
    Stage<T>& st = stages[sidx];
    const TileRef cur = sh_tile[it & 1];
    const BwdDesc& d = bt.d[cur.di];

    // Producer: next tile into the other stage (freed by the barrier that
    // ended the previous iteration).
    const uint32_t next_id = tile_id + gridDim.x;
    if (tid == 0 && next_id < total) {
      bulk_wait_read_all();  // the stage's last bulk store has read it
      const TileRef nxt = locate_full<T>(bt, next_id);
      sh_tile[(it + 1) & 1] = nxt;
      if (bt.d[nxt.di].vec) issue_tile<T>(bt.d[nxt.di], nxt, stages[sidx ^ 1], &bars[sidx ^ 1]);
    }

    const uint64_t w0 = cur.w0, w1 = cur.w1;
    const int off = cur.off;  // tile start in stage
    if (d.vec) {
      mbar_wait(&bars[sidx], (phase_bits >> sidx) & 1u);
      phase_bits ^= 1u << sidx;
      // elements past the bulk window (only at the very end of a tensor)
      const uint64_t e_end = cur.A + (uint64_t)cur.m;
      const uint64_t e_w1 = w1 / sizeof(T);
      if (e_w1 < e_end) {
        for (uint64_t e = e_w1 + tid; e < e_end; e += kBwdThreads) {
          st.x[e - w0 / sizeof(T)] = static_cast<const T*>(d.x)[e];
          st.up[e - w0 / sizeof(T)] = static_cast<const T*>(d.up)[e];
        }
        __syncthreads();
      }
    } else {
      for (int e = tid; e < cur.m; e += kBwdThreads) {
        st.x[off + e] = static_cast<const T*>(d.x)[cur.A + e];
        st.up[off + e] = static_cast<const T*>(d.up)[cur.A + e];
      }
      __syncthreads();
    }

    // This thread's leaf group: two left folds from 0.0 over its halves (or
    // one fold if <= 8 elements), in registers, then their sum.
    int glo, glen;
    gc.get(cur.m, (int)d.g, tid, glo, glen);
    DivCtx dc;
    dc.s = pin(cur.s);
    dc.y = pin(cur.y);
    dc.usable = cur.s >= 0x1p-100 && cur.s <= 0x1p100;
    const double q = pin(d.q);
    const bool want_dx = d.dx != nullptr;
    T* sx = st.x + off + glo;
    const T* su = st.up + off + glo;
    const double v = want_dx ? group_sum<T, true>(sx, su, glen, dc, q)
                             : group_sum<T, false>(sx, su, glen, dc, q);
    __syncthreads();  // stage.x now holds d_input for the whole tile

    // Warp-level butterfly now; the cross-warp step after the copy-out.
    const int groups = 1 << d.g;
    const int wl = groups < 32 ? groups : 32;
    double wv = v;
    for (int o = 1; o < wl; o <<= 1) wv = __dadd_rn(wv, __shfl_xor_sync(0xffffffffu, wv, o));
    if ((tid & 31) == 0) red[tid >> 5] = wv;

    // d_input -> HBM. The 16-byte-aligned interior of the tile goes out as
    // ONE bulk store (TMA) issued by thread 0 after the barrier below; the
    // ragged head/tail elements are stored by threads.
    const uint64_t b0 = cur.A * sizeof(T), b1 = (cur.A + (uint64_t)cur.m) * sizeof(T);
    const uint64_t i0 = (b0 + 15) & ~uint64_t(15), i1 = b1 & ~uint64_t(15);
    if (want_dx) {
      const int head = (int)((i0 > b1 ? b1 : i0) - b0) / (int)sizeof(T);
      const int tail0 = i1 > i0 ? (int)((i1 - b0) / sizeof(T)) : head;
      for (int e = tid; e < head; e += kBwdThreads)
        static_cast<T*>(d.dx)[cur.A + e] = st.x[off + e];
      for (int e = tail0 + tid; e < cur.m; e += kBwdThreads)
        static_cast<T*>(d.dx)[cur.A + e] = st.x[off + e];
    }
    __syncthreads();  // d_input complete in the stage; red complete
    if (tid == 0 && want_dx && i1 > i0) {
      fence_proxy_async_smem();  // generic-proxy smem writes -> async proxy
      bulk_s2g(static_cast<char*>(d.dx) + i0, reinterpret_cast<const char*>(st.x) + (i0 - w0),
               (uint32_t)(i1 - i0));
      bulk_commit();
    }

    // Perfect-tree combine of the warp sums (groups > 32) -> tile partial.
    if (tid < 32) {
      const int nw = groups > 32 ? groups >> 5 : 1;
      double r = tid < nw ? red[tid] : 0.0;
      for (int o = 1; o < nw; o <<= 1) r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, o));
      if (tid == 0) d.partials[((uint64_t)cur.seg << d.tps_log) + cur.t] = r;
    }
  }
  if (tid == 0) bulk_wait_all();  // d_input bulk stores complete before exit
}

// Finisher: one warp per (descriptor, channel). Each row's 2^tps_log tile
// partials are reduced in perfect-tree order (lane slices + xor butterfly),
// times chain[c]; rows of the channel are folded in row order.
constexpr int kFinSmem = 4096;  // partials per row staged in smem (32 KB)

__global__ void __launch_bounds__(32) bwd_finish_kernel(const __grid_constant__ BwdBatch bt,
                                                        uint32_t warp_base_mul) {
  __shared__ double sp[kFinSmem];
  // locate (descriptor, channel) of this warp: warps are laid out per
  // descriptor as chans consecutive warps
  uint32_t w = blockIdx.x;
  int di = 0;
  while (di < bt.n && w >= bt.d[di].chans) {
    w -= bt.d[di].chans;
    ++di;
  }
  if (di >= bt.n) return;
  const BwdDesc& d = bt.d[di];
  const uint32_t c = w;
  const int lane = threadIdx.x;
  const uint32_t tps = 1u << d.tps_log;
  const uint32_t lanes = tps < 32u ? tps : 32u;
  const uint32_t per = tps / lanes;
  const double chain = d.chain[c];
  double acc = 0.0;
  for (uint32_t o = 0; o < d.outer; ++o) {
    const double* p = d.partials + (((uint64_t)o * d.chans + c) << d.tps_log);
    double v = 0.0;
    if (per == 1) {
      v = (uint32_t)lane < lanes ? p[lane] : 0.0;
    } else if (tps <= (uint32_t)kFinSmem) {
      for (uint32_t i = lane; i < tps; i += 32) sp[i] = p[i];
      __syncwarp();
      double* mine = sp + (uint32_t)lane * per;
      for (uint32_t width = per; width > 1; width >>= 1)
        for (uint32_t k = 0; k < width / 2; ++k) mine[k] = __dadd_rn(mine[2 * k], mine[2 * k + 1]);
      v = mine[0];
      __syncwarp();
    } else {
      // huge rows: in place over the lane's own global slice
      double* mine = const_cast<double*>(p) + (uint64_t)lane * per;
      for (uint32_t width = per; width > 1; width >>= 1)
        for (uint32_t k = 0; k < width / 2; ++k) mine[k] = __dadd_rn(mine[2 * k], mine[2 * k + 1]);
      v = mine[0];
    }
    for (uint32_t off = 1; off < lanes; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    const double r = __dmul_rn(v, chain);
    // accumulate == 0: ((r0 + r1) + ...); else ((d_log_s + r0) + r1) + ...
    if (o == 0) acc = d.accumulate ? __dadd_rn(d.d_log_s[c], r) : r;
    else acc = __dadd_rn(acc, r);
  }
  if (lane == 0) d.d_log_s[c] = acc;
  (void)warp_base_mul;
}

template <typename T>
constexpr size_t stage_bytes() {
  return sizeof(Stage<T>) * kStages;
}

}  // namespace

cudaError_t bwd_occupancy(int dtype, int* blocks_per_sm) {
  cudaError_t e;
  if (dtype == 0) {
    e = cudaFuncSetAttribute(bwd_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)stage_bytes<float>());
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, bwd_kernel<float>,
                                                         kBwdThreads, stage_bytes<float>());
  }
  e = cudaFuncSetAttribute(bwd_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)stage_bytes<__half>());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, bwd_kernel<__half>,
                                                       kBwdThreads, stage_bytes<__half>());
}

cudaError_t launch_bwd(int dtype, const BwdBatch& b, int grid, cudaStream_t st) {
  const uint32_t tiles = b.tile_begin[b.n];
  if (tiles == 0) return cudaSuccess;
  if ((uint32_t)grid > tiles) grid = (int)tiles;
  if (dtype == 0)
    bwd_kernel<float><<<grid, kBwdThreads, stage_bytes<float>(), st>>>(b);
  else
    bwd_kernel<__half><<<grid, kBwdThreads, stage_bytes<__half>(), st>>>(b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  uint32_t warps = 0;
  for (int i = 0; i < b.n; ++i) warps += b.d[i].chans;
  bwd_finish_kernel<<<warps, 32, 0, st>>>(b, 0u);
  return cudaGetLastError();
}

}  // namespace qfb
