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
//             mbarrier ring, 2..8 stages); each consumer thread owns one leaf
//             group, computes its elements' terms in registers and folds them
//             in reference order, writing d_input back into the stage; the
//             producer warp reduces the 2^g group sums as a perfect tree
//             (lane subtrees + xor butterfly = the tile's subtree sum) and
//             sends d_input out with one TMA bulk store;
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
#include <stdlib.h>

#include "qfb_device.cuh"
#include "qfb_kernels.h"

namespace qfb {

namespace {

constexpr int kMaxStages = 8;
// Probe variants (template V, QFB_BWD_VARIANT): memory pipeline only (no
// arithmetic, d_input = staged x) / arithmetic only (tiles loaded once,
// no refills or stores). Not used in production; results in DESIGN.md §7.
constexpr int kProbeNoCompute = 8;
constexpr int kProbeNoLoads = 16;
// Consumer-side tree (production when every row has full 256-group
// tiles): each consumer warp reduces its 32 group sums with a 5-level xor
// butterfly (a perfect subtree: the node at depth D - 5) and leaves the
// sum in shared memory; the producer combines the tile's 8 warp sums
// (3-level butterfly over lanes 0..7) into the tile partial. Before, the
// producer folded all 256 group sums itself (8 per lane + 5 levels) on the
// refill path of every tile.
constexpr int kWarpPart = 32;

constexpr int kWinPad = 32;                // window slack: 16-byte rounding at both ends
constexpr size_t kRingBudget = 76 * 1024;  // default per-CTA ring + sums: 3 CTAs per SM
// group sums of one stage use, double-buffered per stage (the producer reads
// use u's sums after it has already refilled the stage for use u + 1)
constexpr size_t kRedBytes = 2 * kBwdThreads * sizeof(double);
constexpr size_t kSmemMax = 220 * 1024;    // dynamic smem attribute (ring + sums; + static <= 227 KB)

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

// One ring stage: the x and upstream windows of a tile (runtime stride).
template <typename T>
struct Stage {
  T* x;
  T* up;
};

template <typename T>
__device__ __forceinline__ Stage<T> stage_at(unsigned char* base, uint32_t stage_elems, int s) {
  T* p = reinterpret_cast<T*>(base) + (size_t)s * 2 * stage_elems;
  return Stage<T>{p, p + stage_elems};
}

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
  float hthr;   // kHalfF32: binary16 clip threshold (half_clip_threshold), per tile
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
// L2 hints (QFB_L2_HINTS mask, A/B): 2 = x loads evict_last, 4 = upstream
// loads evict_first, 8 = d_input stores evict_first
__constant__ int c_bwd_l2_hints = 0;

template <typename T>
__device__ __forceinline__ void issue_tile(const BwdDesc& d, const TileRef& r, Stage<T>& st,
                                           uint64_t* bar) {
  const uint32_t bytes = (uint32_t)(r.w1 - r.w0);
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(bar, 2 * bytes);
  if (bytes) {
    const int h = c_bwd_l2_hints;
    if (h & 2) bulk_g2s_hint(st.x, static_cast<const char*>(d.x) + r.w0, bytes, bar, l2_evict_last());
    else bulk_g2s(st.x, static_cast<const char*>(d.x) + r.w0, bytes, bar);
    if (h & 4) bulk_g2s_hint(st.up, static_cast<const char*>(d.up) + r.w0, bytes, bar, l2_evict_first());
    else bulk_g2s(st.up, static_cast<const char*>(d.up) + r.w0, bytes, bar);
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
// Exact reference semantics for the rare elements the fast path does not
// cover (inf/NaN operands, scales outside [2^-100, 2^100]): IEEE division,
// quant.hpp:217-228 verbatim. Out of line so it never bloats the hot loop.
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

// Fast-path terms of one element, no branches: term, d_input (finite
// upstream) and whether the fast path applies (else: slow_elem).
struct FastTerm {
  double term;
  float dx;
  bool ok;
};

__device__ __forceinline__ FastTerm fast_elem(float xv, float uv, const DivCtx& dc, double q) {
  FastTerm f;
  const bool up_finite = (__float_as_uint(uv) & 0x7f800000u) != 0x7f800000u;
  // correctly rounded for every finite x (markstein2_div; x = +-0 gives a
  // zero whose sign d_ds = rint(z) - z = +0 does not observe); only inf/NaN
  // operands and scales outside [2^-100, 2^100] take the IEEE path
  const double z = markstein2_div((double)xv, dc);
  f.ok = dc.usable && fabsf(xv) <= 3.402823466e38f && up_finite;
  const bool mask = fabs(z) <= q;
  const double d_ds = mask ? __dadd_rn(rint(z), -z) : copysign(q, z);
  f.term = __dmul_rn(d_ds, (double)uv);
  f.dx = mask ? uv : __uint_as_float(__float_as_uint(uv) & 0x80000000u);
  return f;
}

__device__ __forceinline__ void fix_slow(FastTerm& f, float xv, float uv, double s, double q) {
  if (!f.ok) {
    const double2 r = slow_elem(xv, uv, s, q);
    f.term = r.x;
    f.dx = (float)r.y;  // exact: r.y is a float widened
  }
}

// One element: term = d_ds * up (double) and d_input, with z = RN(x/s)
// from markstein2_div (qfb_device.cuh); inf/NaN operands take the exact
// IEEE path in slow_elem (returned in registers, never via memory).
template <typename T, bool kDx>
__device__ __forceinline__ double elem(T* sx, const T* su, int k, const DivCtx& dc, double q) {
  const float xv = to_f<T>(sx[k]);
  const float uv = to_f<T>(su[k]);
  FastTerm f = fast_elem(xv, uv, dc, q);
  fix_slow(f, xv, uv, dc.s, q);
  if (kDx) sx[k] = from_f<T>(f.dx);
  return f.term;
}

// A leaf group's sum in the reference order: fold(left half) + fold(right
// half) from 0.0 each (or one fold if <= 8 elements). Generic sizes; the
// two folds are independent chains, interleaved for ILP.
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
#pragma unroll 2
  for (int k = 0; k < h; ++k) {
    const double tl = elem<T, kDx>(sx, su, k, dc, q);
    const double tr = elem<T, kDx>(rx, ru, k, dc, q);
    acc_l = __dadd_rn(acc_l, tl);
    acc_r = __dadd_rn(acc_r, tr);
  }
  if (glen - h > h) acc_r = __dadd_rn(acc_r, elem<T, kDx>(rx, ru, h, dc, q));
  return __dadd_rn(acc_l, acc_r);
}

// Unchecked fast path for tiles with a usable scale (s in [2^-100, 2^100]):
// no per-element inf/NaN test. It is exact for every operand:
//  - non-finite x: markstein2_div gives NaN, so mask = false as for the IEEE
//    quotient (inf or NaN), and the saturated term takes its sign from x
//    (x > 0 ? q : -q), which is the reference's (z > 0 ? q : -q) for
//    z = x/s = +-inf or NaN;
//  - non-finite upstream: the term d_ds * up is the reference's product
//    (d_ds is finite here); only d_input differs (masked NaN / inf rules),
//    and such an element makes the group sum non-finite (term = inf or
//    NaN; a finite term is < 2^136), so one test per group finds it and
//    fix_nonfinite_up rewrites those d_input values.
// rint(z) for |z| < 2^51 (every z with |z| <= q): RN(z + 1.5*2^52) lies in
// (2^52, 2^53) where the spacing is 1, so the add rounds z to the nearest
// integer, ties to even, and the subtraction is exact. Two DADDs on the
// FP64 pipe instead of FRND.F64 on the quarter-rate XU pipe; identical bits
// to rint(z) - z, including the +0 of integer z.
__device__ __forceinline__ double rint_small(double z) {
  return __dadd_rn(__dadd_rn(z, 0x1.8p52), -0x1.8p52);
}

// Arithmetic options of the fast path (template M): kMathMagic = rint by
// rint_small, kMathDD = quotient by markstein_dd. Bit-identical results.
constexpr int kMathMagic = 1;
constexpr int kMathDD = 2;
constexpr int kMathSel = 4;  // word-wise term select (select_term)

template <int M>
__device__ __forceinline__ double quotient(double x, const DivCtx& dc) {
  return (M & kMathDD) ? markstein_dd(x, dc) : markstein2_div(x, dc);
}

// d_ds = mask ? rint(z) - z : (x > 0 ? q : -q), selected word by word: q
// is an integer <= 32767, so the low word of +-q is 0 and its high word
// differs from q's only in the sign bit (three integer selects instead of
// four FSELs of the two double selects). Used by the binary16 terms (f16
// step 0.1185 -> 0.1156 ms, r02bl); the f32 terms keep the double selects.
__device__ __forceinline__ double select_term(bool mask, double dd, bool pos, double q) {
  const int qh = __double2hiint(q);
  const int sh = pos ? qh : (int)((unsigned)qh | 0x80000000u);
  return __hiloint2double(mask ? __double2hiint(dd) : sh, mask ? __double2loint(dd) : 0);
}

template <int M = 0>
__device__ __forceinline__ double fast_term(float xv, float uv, const DivCtx& dc, double q,
                                            float& dx) {
  const double z = quotient<M>((double)xv, dc);
  const bool mask = fabs(z) <= q;
  const double r = (M & kMathMagic) ? rint_small(z) : rint(z);
  // (select_term measured slower here: f32 step 0.1336 -> 0.1352 ms, r02bl)
  const double d_ds = mask ? __dadd_rn(r, -z) : (xv > 0.0f ? q : -q);
  dx = mask ? uv : __uint_as_float(__float_as_uint(uv) & 0x80000000u);
  return __dmul_rn(d_ds, (double)uv);
}

// binary16 operands: converted straight to double (one F2F.F64.F16 each,
// exact) and d_input written from up's storage bits (mask ? up : +-0 with
// up's sign, exact for finite up; non-finite up is fixed per group as for
// f32). Same values as fast_term on the widened floats.
__device__ __forceinline__ double h2d(__half h) {
  double d;
  asm("cvt.f64.f16 %0, %1;" : "=d"(d) : "h"(__half_as_ushort(h)));
  return d;
}
template <int M = 0>
__device__ __forceinline__ double fast_term_h(__half xh, __half uh, const DivCtx& dc, double q,
                                              __half* dx) {
  const double xd = h2d(xh);
  const double z = quotient<M>(xd, dc);
  const bool mask = fabs(z) <= q;
  const double r = (M & kMathMagic) ? rint_small(z) : rint(z);
  const double d_ds = (M & kMathSel) ? select_term(mask, __dadd_rn(r, -z), xd > 0.0, q)
                                     : (mask ? __dadd_rn(r, -z) : (xd > 0.0 ? q : -q));
  if (dx) {
    const unsigned short b = __half_as_ushort(uh);
    *dx = __ushort_as_half(mask ? b : (unsigned short)(b & 0x8000u));
  }
  return __dmul_rn(d_ds, h2d(uh));
}

// d_input of the group's non-finite upstream values (rare): the fast path
// stored up (mask) or +-0 (masked out); masked_upstream gives the
// reference's value from that mask.
template <typename T>
static __device__ __noinline__ void fix_nonfinite_up(T* sx, const T* su, int glen) {
  for (int k = 0; k < glen; ++k) {
    const float uv = to_f<T>(su[k]);
    if ((__float_as_uint(uv) & 0x7f800000u) == 0x7f800000u) {
      const bool mask = isinf(to_f<T>(sx[k]));
      sx[k] = from_f<T>(masked_upstream(mask, uv));
    }
  }
}

template <typename T, bool kDx, int LR, int M = 0>
__device__ __forceinline__ double group_sum_lr_u(T* sx, const T* su, int h, const DivCtx& dc,
                                                 double q) {
  T* rx = sx + h;
  const T* ru = su + h;
  const bool lv = h == LR;
  double acc_l = 0.0, acc_r = 0.0;
#pragma unroll
  for (int k = 0; k < LR; ++k) {
    const bool l0 = k < LR - 1 || lv;  // left slot k valid
    double t0, t2;
    if constexpr (sizeof(T) == 2) {
      t0 = l0 ? fast_term_h<M>(sx[k], su[k], dc, q, kDx ? sx + k : nullptr) : 0.0;
      t2 = fast_term_h<M>(rx[k], ru[k], dc, q, kDx ? rx + k : nullptr);
    } else {
      const float x0 = l0 ? to_f<T>(sx[k]) : 0.0f, u0 = l0 ? to_f<T>(su[k]) : 0.0f;
      const float x2 = to_f<T>(rx[k]), u2 = to_f<T>(ru[k]);
      float d0, d2;
      t0 = fast_term<M>(x0, u0, dc, q, d0);
      t2 = fast_term<M>(x2, u2, dc, q, d2);
      if (kDx) {
        if (l0) sx[k] = from_f<T>(d0);
        rx[k] = from_f<T>(d2);
      }
    }
    if (l0) acc_l = __dadd_rn(acc_l, t0);
    acc_r = __dadd_rn(acc_r, t2);
  }
  const double v = __dadd_rn(acc_l, acc_r);
  if (kDx && __builtin_expect((__double2hiint(v) & 0x7ff00000) == 0x7ff00000, 0))
    fix_nonfinite_up<T>(sx, su, h + LR);
  return v;
}

// Dispatch on the right-half length (groups of 9..16 elements, the only
// sizes of rows with >= 16 * 2^g elements); other sizes take the generic loop.
template <typename T, bool kDx, int M = 0>
__device__ __forceinline__ double group_sum_any(T* sx, const T* su, int glen, const DivCtx& dc,
                                                double q) {
  if (glen >= 9 && dc.usable) {
    const int lr = (glen + 1) >> 1, h = glen >> 1;
    switch (lr) {
      case 5: return group_sum_lr_u<T, kDx, 5, M>(sx, su, h, dc, q);
      case 6: return group_sum_lr_u<T, kDx, 6, M>(sx, su, h, dc, q);
      case 7: return group_sum_lr_u<T, kDx, 7, M>(sx, su, h, dc, q);
      default: return group_sum_lr_u<T, kDx, 8, M>(sx, su, h, dc, q);
    }
  }
  return group_sum<T, kDx>(sx, su, glen, dc, q);  // short groups / unusable scales: checked
}

// ---------------------------------------------------------------------
// Quad consumer (kQuad): 4 consumer warps, each lane owns TWO adjacent leaf
// groups of the tile (2t, 2t+1: the children of node t at depth g - 1), so
// four fold chains (left/right half of each group) run interleaved per lane
// and the per-tile work of a warp (barrier wait, descriptor reads, tree
// butterfly, handoff) is spread over twice the elements. The lane's two
// group sums form their parent node (A + B); a 5-level xor butterfly gives
// the warp's 64-group subtree, and the producer combines the 4 warp sums.
// ---------------------------------------------------------------------
struct PairCache {
  int k0 = -1, lo0 = 0, m0 = 0;
  int k1 = -1, lo1 = 0, m1 = 0;
  // parent node of lane pair t (path t, g - 1 levels) in a tile of m elements
  __device__ __forceinline__ void get(int m, int g, int t, int& plo, int& pm) {
    const int k = m | (g << 16);
    if (k0 == k) {
      plo = lo0;
      pm = m0;
      return;
    }
    if (k1 == k) {
      plo = lo1;
      pm = m1;
      return;
    }
    int l = 0, mm = m;
    descend<int>(l, mm, (uint32_t)t, g - 1);
    k1 = k0;
    lo1 = lo0;
    m1 = m0;
    k0 = k;
    lo0 = l;
    m0 = mm;
    plo = l;
    pm = mm;
  }
};

// One fold slot of a half-group: term of element k (predicated on `on`),
// d_input written back in place when kDx.
template <typename T, bool kDx, int M>
__device__ __forceinline__ void quad_slot(T* px, const T* pu, int k, bool on, const DivCtx& dc, double q,
                                          double& acc) {
  double t;
  if constexpr (sizeof(T) == 2) {
    t = fast_term_h<M>(px[k], pu[k], dc, q, (kDx && on) ? px + k : nullptr);
  } else {
    float d;
    t = fast_term<M>(on ? px[k] : 0.0f, on ? pu[k] : 0.0f, dc, q, d);
    if (kDx && on) px[k] = d;
  }
  if (on) acc = __dadd_rn(acc, t);
}

// Sums of two sibling leaf groups A = [0, la), B = [la, la + lb) (9..16
// elements each, lb - la in {0, 1}) in the reference order, four chains
// interleaved: fold(A left) + fold(A right), fold(B left) + fold(B right).
// LR = the longest half; only the last two slots can be short.
template <typename T, bool kDx, int M, int LR>
__device__ __forceinline__ double quad_sum_u(T* sx, const T* su, int la, int lb, const DivCtx& dc, double q) {
  const int ha = la >> 1, hb = lb >> 1;
  const int ra = la - ha, rb = lb - hb;
  T* ax = sx;
  T* arx = sx + ha;
  T* bx = sx + la;
  T* brx = sx + la + hb;
  const T* au = su;
  const T* aru = su + ha;
  const T* bu = su + la;
  const T* bru = su + la + hb;
  double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
  for (int k = 0; k < LR; ++k) {
    const bool tail = k >= LR - 2;
    quad_slot<T, kDx, M>(ax, au, k, !tail || k < ha, dc, q, a0);
    quad_slot<T, kDx, M>(arx, aru, k, !tail || k < ra, dc, q, a1);
    quad_slot<T, kDx, M>(bx, bu, k, !tail || k < hb, dc, q, b0);
    quad_slot<T, kDx, M>(brx, bru, k, !tail || k < rb, dc, q, b1);
  }
  const double va = __dadd_rn(a0, a1);
  const double vb = __dadd_rn(b0, b1);
  if (kDx && __builtin_expect((__double2hiint(va) & 0x7ff00000) == 0x7ff00000, 0)) fix_nonfinite_up<T>(sx, su, la);
  if (kDx && __builtin_expect((__double2hiint(vb) & 0x7ff00000) == 0x7ff00000, 0))
    fix_nonfinite_up<T>(sx + la, su + la, lb);
  return __dadd_rn(va, vb);
}

template <typename T, bool kDx, int M>
__device__ __forceinline__ double quad_sum(T* sx, const T* su, int pm, const DivCtx& dc, double q) {
  const int la = pm >> 1, lb = pm - la;
  if (la >= 9 && dc.usable) {
    const int lr = ((lb + 1) >> 1) > ((la + 1) >> 1) ? ((lb + 1) >> 1) : ((la + 1) >> 1);
    switch (lr) {
      case 5: return quad_sum_u<T, kDx, M, 5>(sx, su, la, lb, dc, q);
      case 6: return quad_sum_u<T, kDx, M, 6>(sx, su, la, lb, dc, q);
      case 7: return quad_sum_u<T, kDx, M, 7>(sx, su, la, lb, dc, q);
      default: return quad_sum_u<T, kDx, M, 8>(sx, su, la, lb, dc, q);
    }
  }
  // short groups / unusable scales: the checked per-group path
  const double va = group_sum<T, kDx>(sx, su, la, dc, q);
  const double vb = group_sum<T, kDx>(sx + la, su + la, lb, dc, q);
  return __dadd_rn(va, vb);
}

// ---------------------------------------------------------------------
// binary16 storage with float32 terms (opt-in: QFB_OPT_BWD_HALF_FP32).
// The scale-gradient terms are computed in float32 instead of the
// reference's binary64, so d_log_s agrees with the reference within the
// FP16 tolerance of north_star (measured ~1e-6 relative, bound stated in
// DESIGN.md) rather than bitwise; d_input stays bitwise because the clip
// mask is decided exactly:
//  - mask: |RN64(x/s)| <= q  <=>  |x| <= T, T the largest binary16 value
//    with RN64(T/s) <= q (RN64(h/s) is monotone in h), found per tile with
//    the exact double quotient;
//  - z = x/s as a float pair p + zl from a float pair reciprocal (yh + yl =
//    RN(1/s) to ~2^-48): p = RN(x*yh), zl = RN(fma(x, yh, -p) + x*yl) — the
//    product error is exact, so p + zl is x/s within ~2^-45 relative;
//  - d = (rint(p) - p) - zl, wrapped into [-1/2, 1/2] (d - rint(d)): the
//    nearest integer of p + zl, not of p, so a quotient just past a
//    half-integer does not flip d by 1 (that flip would cost |up| in the sum);
//  - term = d * up (clipped: +-q * up, exact), folded in float32 per leaf
//    group in the reference order, widened to double per group (one F2F per
//    group instead of two per element), and the tree above in double.
// Four fold chains per lane (quad layout), short FP32 latencies: the pass
// is bound by the memory pipeline instead of FP64/XU latency.
// ---------------------------------------------------------------------
struct HalfCtx {
  float yh, yl;  // float pair of RN(1/s)
  float t;       // clip threshold on |x| (a binary16 value)
  float q;
};

// Largest binary16 h >= 0 with RN64(h/s) <= q (exact double quotient).
__device__ __forceinline__ float half_clip_threshold(const DivCtx& dc, double q) {
  const double t = q * dc.s;
  unsigned short h = __half_as_ushort(__float2half_rd(__double2float_rd(t)));
  if (h >= 0x7c00u) h = 0x7bffu;
  auto ok = [&](unsigned short b) {
    return fabs(markstein_dd((double)__half2float(__ushort_as_half(b)), dc)) <= q;
  };
  while (h < 0x7bffu && ok((unsigned short)(h + 1))) ++h;
  while (h > 0u && !ok(h)) --h;
  return __half2float(__ushort_as_half(h));
}

// thr: half_clip_threshold(dc, q), computed per tile by the producer
__device__ __forceinline__ HalfCtx make_half_ctx(const DivCtx& dc, double q, float thr) {
  HalfCtx h;
  h.yh = (float)dc.y;
  h.yl = (float)(dc.y - (double)h.yh);
  h.t = thr;
  h.q = (float)q;
  return h;
}

template <bool kDx>
__device__ __forceinline__ void h32_slot(__half* px, const __half* pu, int k, bool on, const HalfCtx& hc,
                                         float& acc) {
  const float x = __half2float(px[k]);
  const float u = __half2float(pu[k]);
  const bool mask = fabsf(x) <= hc.t;
  const float p = __fmul_rn(x, hc.yh);
  const float zl = __fmaf_rn(x, hc.yl, __fmaf_rn(x, hc.yh, -p));
  // rint by the float magic number 1.5*2^23 (exact for |v| < 2^22, i.e. for
  // every unclipped p and for d): two FADDs on the FMA pipe, not FRND on XU
  constexpr float kM = 12582912.0f;
  float d = __fsub_rn(__fsub_rn(__fsub_rn(__fadd_rn(p, kM), kM), p), zl);
  d = __fsub_rn(d, __fsub_rn(__fadd_rn(d, kM), kM));
  const float sat = x > 0.0f ? hc.q : -hc.q;
  const float t = __fmul_rn(mask ? d : sat, u);
  if (kDx && on) {
    const unsigned short b = __half_as_ushort(pu[k]);
    px[k] = __ushort_as_half(mask ? b : (unsigned short)(b & 0x8000u));
  }
  if (on) acc = __fadd_rn(acc, t);
}

template <bool kDx, int LR>
__device__ __forceinline__ double quad_sum_h32_u(__half* sx, const __half* su, int la, int lb, const HalfCtx& hc) {
  const int ha = la >> 1, hb = lb >> 1;
  const int ra = la - ha, rb = lb - hb;
  float a0 = 0.0f, a1 = 0.0f, b0 = 0.0f, b1 = 0.0f;
#pragma unroll
  for (int k = 0; k < LR; ++k) {
    const bool tail = k >= LR - 2;
    h32_slot<kDx>(sx, su, k, !tail || k < ha, hc, a0);
    h32_slot<kDx>(sx + ha, su + ha, k, !tail || k < ra, hc, a1);
    h32_slot<kDx>(sx + la, su + la, k, !tail || k < hb, hc, b0);
    h32_slot<kDx>(sx + la + hb, su + la + hb, k, !tail || k < rb, hc, b1);
  }
  const double va = __dadd_rn((double)a0, (double)a1);
  const double vb = __dadd_rn((double)b0, (double)b1);
  if (kDx && __builtin_expect((__double2hiint(va) & 0x7ff00000) == 0x7ff00000, 0)) fix_nonfinite_up<__half>(sx, su, la);
  if (kDx && __builtin_expect((__double2hiint(vb) & 0x7ff00000) == 0x7ff00000, 0))
    fix_nonfinite_up<__half>(sx + la, su + la, lb);
  return __dadd_rn(va, vb);
}

// Sum of two sibling leaf groups with float32 terms (usable scales, groups
// of >= 9 elements); other cases take the exact double path.
template <bool kDx>
__device__ __forceinline__ double quad_sum_h32(__half* sx, const __half* su, int pm, const DivCtx& dc, double q,
                                               const HalfCtx& hc) {
  const int la = pm >> 1, lb = pm - la;
  if (la >= 9 && dc.usable) {
    const int lr = ((lb + 1) >> 1) > ((la + 1) >> 1) ? ((lb + 1) >> 1) : ((la + 1) >> 1);
    switch (lr) {
      case 5: return quad_sum_h32_u<kDx, 5>(sx, su, la, lb, hc);
      case 6: return quad_sum_h32_u<kDx, 6>(sx, su, la, lb, hc);
      case 7: return quad_sum_h32_u<kDx, 7>(sx, su, la, lb, hc);
      default: return quad_sum_h32_u<kDx, 8>(sx, su, la, lb, hc);
    }
  }
  const double va = group_sum<__half, kDx>(sx, su, la, dc, q);
  const double vb = group_sum<__half, kDx>(sx + la, su + la, lb, dc, q);
  return __dadd_rn(va, vb);
}

// ---------------------------------------------------------------------
// Warp-specialized main pass. 8 consumer warps (256 lanes = 256 leaf
// groups of a tile) + 1 producer warp. Per stage s of the 2-deep ring:
//   full[s]  producer -> consumers: TileRef written, x/up landed (TMA tx)
//   done[s]  consumers -> producer: d_input written into the stage and the
//            8 warp sums in red[s] (one arrive per consumer warp)
// The producer finalizes tile j (cross-warp tree step -> partial, ragged
// d_input ends, one TMA bulk store of the aligned interior), waits for the
// store to have read the stage, then refills the stage with tile j+2.
// Consumers never execute a CTA-wide barrier.
// ---------------------------------------------------------------------
constexpr int kConsumerWarps = kBwdThreads / 32;      // 8
constexpr int kQuad = 64;         // 4 consumer warps x 2 leaf groups per lane (see quad_sum)
constexpr int kMagicRint = 256;   // rint via rint_small (FP64 pipe) instead of FRND (XU pipe)
constexpr int kDDiv = 2048;       // quotient via markstein_dd (4 FP64 ops) instead of markstein2_div (5)
constexpr int kHalfF32 = 4096;    // binary16 storage, float32 terms (QFB_OPT_BWD_HALF_FP32)
constexpr int kL2Pre = 8192;      // producer prefetches the tile after the next refill into L2
template <int V>
__host__ __device__ constexpr int math_of() {
  return ((V & kMagicRint) ? kMathMagic : 0) | ((V & kDDiv) ? kMathDD : 0) | kMathSel;
}
template <int V>
__host__ __device__ constexpr int cons_warps() { return (V & kQuad) ? 4 : kConsumerWarps; }
template <int V>
__host__ __device__ constexpr int cta_threads() { return cons_warps<V>() * 32 + 32; }

__device__ __forceinline__ TileRef shfl_ref(const TileRef& r, int src) {
  constexpr unsigned kAll = 0xffffffffu;
  TileRef o;
  o.di = __shfl_sync(kAll, r.di, src);
  o.seg = __shfl_sync(kAll, r.seg, src);
  o.t = __shfl_sync(kAll, r.t, src);
  o.c = __shfl_sync(kAll, r.c, src);
  o.A = __shfl_sync(kAll, (unsigned long long)r.A, src);
  o.m = __shfl_sync(kAll, r.m, src);
  o.off = __shfl_sync(kAll, r.off, src);
  o.w0 = __shfl_sync(kAll, (unsigned long long)r.w0, src);
  o.w1 = __shfl_sync(kAll, (unsigned long long)r.w1, src);
  o.s = __shfl_sync(kAll, r.s, src);
  o.y = __shfl_sync(kAll, r.y, src);
  o.hthr = __shfl_sync(kAll, r.hthr, src);
  return o;
}

// Stage fill for tile r (r valid on lane 0, computed by locate_full ahead of
// time so no global-memory latency sits between a stage's release and its
// refill).
template <typename T, int V = 0>
__device__ __forceinline__ void produce(const BwdBatch& bt, const TileRef& r, Stage<T>& st,
                                        TileRef* ref, uint64_t* full, int lane,
                                        bool prologue_done = false) {
  // broadcast the fields the lanes need for a manual fill
  const int di = __shfl_sync(0xffffffffu, r.di, 0);
  const BwdDesc& d = bt.d[di];
  if (d.vec) {
    if (lane == 0) {
      *ref = r;
      const uint64_t e_end = r.A + (uint64_t)r.m;
      const uint64_t e_w1 = r.w1 / sizeof(T);
      // elements past the bulk window (only at the very end of a tensor)
      for (uint64_t e = e_w1; e < e_end; ++e) {
        st.x[e - r.w0 / sizeof(T)] = static_cast<const T*>(d.x)[e];
        st.up[e - r.w0 / sizeof(T)] = static_cast<const T*>(d.up)[e];
      }
      if ((V & kProbeNoLoads) && prologue_done) mbar_arrive_expect_tx(full, 0);
      else issue_tile<T>(d, r, st, full);  // arrive.expect_tx releases the stores above
    }
  } else {
    // unaligned buffers: the producer warp fills the stage itself
    const uint64_t A = __shfl_sync(0xffffffffu, r.A, 0);
    const int m = __shfl_sync(0xffffffffu, r.m, 0);
    const int off = __shfl_sync(0xffffffffu, r.off, 0);
    for (int e = lane; e < m; e += 32) {
      st.x[off + e] = static_cast<const T*>(d.x)[A + e];
      st.up[off + e] = static_cast<const T*>(d.up)[A + e];
    }
    __syncwarp();
    if (lane == 0) {
      *ref = r;
      mbar_arrive_expect_tx(full, 0);
    }
  }
}

// Perfect tree over the tile's 2^g group sums, lane part: each lane folds
// `per` consecutive sums as a perfect subtree (read into registers before
// the stage is refilled); tile_sum() finishes with an xor butterfly.
__device__ __forceinline__ double lane_subtree(const BwdDesc& d, const double* red, int lane) {
  const int groups = 1 << d.g;
  const int per = groups >= 32 ? groups >> 5 : 1;
  const int lanes_used = groups >= 32 ? 32 : groups;
  double r = 0.0;
  if (lane < lanes_used) {
    const double* g = red + lane * per;
    switch (per) {
      case 1: r = g[0]; break;
      case 2: r = __dadd_rn(g[0], g[1]); break;
      case 4: r = __dadd_rn(__dadd_rn(g[0], g[1]), __dadd_rn(g[2], g[3])); break;
      default:
        r = __dadd_rn(__dadd_rn(__dadd_rn(g[0], g[1]), __dadd_rn(g[2], g[3])),
                      __dadd_rn(__dadd_rn(g[4], g[5]), __dadd_rn(g[6], g[7])));
    }
  }
  return r;
}

__device__ __forceinline__ void tile_sum(const BwdDesc& d, const TileRef& cur, double r) {
  const int groups = 1 << d.g;
  const int lanes_used = groups >= 32 ? 32 : groups;
  for (int o = 1; o < lanes_used; o <<= 1) r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0) d.partials[((uint64_t)cur.seg << d.part_log) + cur.t] = r;
}

// d_input of a finished tile: ragged ends by lanes, the aligned interior as
// one TMA bulk store out of the stage.
template <typename T>
__device__ __forceinline__ void store_dx(const BwdDesc& d, const TileRef& cur, Stage<T>& st,
                                         int lane) {
  if (d.dx == nullptr) return;
  if (!d.vec) {  // a buffer off a 16-byte boundary: element stores
    for (int e = lane; e < cur.m; e += 32) static_cast<T*>(d.dx)[cur.A + e] = st.x[cur.off + e];
    return;
  }
  const uint64_t b0 = cur.A * sizeof(T), b1 = (cur.A + (uint64_t)cur.m) * sizeof(T);
  const uint64_t i0 = (b0 + 15) & ~uint64_t(15), i1 = b1 & ~uint64_t(15);
  const int head = (int)(((i0 > b1 ? b1 : i0) - b0) / sizeof(T));
  const int tail0 = i1 > i0 ? (int)((i1 - b0) / sizeof(T)) : head;
  for (int e = lane; e < head; e += 32) static_cast<T*>(d.dx)[cur.A + e] = st.x[cur.off + e];
  for (int e = tail0 + lane; e < cur.m; e += 32) static_cast<T*>(d.dx)[cur.A + e] = st.x[cur.off + e];
  if (lane == 0 && i1 > i0) {
    fence_proxy_async_smem();
    if (c_bwd_l2_hints & 8)
      bulk_s2g_hint(static_cast<char*>(d.dx) + i0, reinterpret_cast<const char*>(st.x) + (i0 - cur.w0),
                    (uint32_t)(i1 - i0), l2_evict_first());
    else
      bulk_s2g(static_cast<char*>(d.dx) + i0, reinterpret_cast<const char*>(st.x) + (i0 - cur.w0),
               (uint32_t)(i1 - i0));
    bulk_commit();
  }
}

// Two CTAs per SM with the registers that frees (more independent
// elements in flight per consumer lane) and a deeper ring (QFB_BWD_CTAS=2).
constexpr int kTwoCtas = 128;

template <typename T, int V>
__global__ void __launch_bounds__(cta_threads<V>(), (V & kTwoCtas) ? 2 : 3) bwd_kernel(const __grid_constant__ BwdBatch bt) {
  constexpr int CW = cons_warps<V>();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ __align__(8) uint64_t done[kMaxStages];
  __shared__ TileRef refs[kMaxStages];
  const int nst = bt.nstages;
  const uint32_t se = bt.stage_elems;
  // per-stage group sums of a tile, after the ring: red[2 * s + parity of
  // the stage's use] (the parity is the stage's full/done phase bit)
  double(*red)[kBwdThreads] = reinterpret_cast<double(*)[kBwdThreads]>(
      smem_raw + (size_t)nst * 2 * se * sizeof(T));
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t total = bt.tile_begin[bt.n];
  pdl_wait();  // the preceding kernel's writes (launch_main) are visible
  if (blockIdx.x >= total) return;

  if (tid == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], CW);
    }
    fence_mbar_init();
    // the finisher (launched as a programmatic dependent) may be scheduled
    // into SM slots as CTAs retire; it waits for this grid's completion
    // (griddepcontrol.wait) before it reads any partial
    pdl_trigger();
  }
  __syncthreads();  // the only CTA barrier: barrier init

  if (warp == CW) {
    // ----------------------------- producer warp -----------------------
    // TileRefs are located 32 at a time (lane i: the CTA's tile ordinal
    // 32*b + i) and broadcast when needed, so the scale load in locate_full
    // costs one memory latency per 32 tiles instead of one per tile.
    TileRef mine;
    uint32_t batch = 0xffffffffu;
    auto ref_of = [&](uint32_t k) -> TileRef {
      const uint32_t b = k >> 5;
      if (b != batch) {
        batch = b;
        const uint32_t id0 = blockIdx.x + ((b << 5) + (uint32_t)lane) * gridDim.x;
        if (id0 < total) {
          const uint32_t id = (bt.layout & kBwdLayoutReverse) ? total - 1u - id0 : id0;
          mine = locate_full<T>(bt, id);
          if constexpr ((V & kHalfF32) != 0) {
            // the fp32-term path's exact clip threshold, once per tile
            DivCtx dc;
            dc.s = mine.s;
            dc.y = mine.y;
            dc.ylo = recip_lo(mine.s, mine.y);
            dc.usable = mine.s >= 0x1p-100 && mine.s <= 0x1p100;
            mine.hthr = dc.usable ? half_clip_threshold(dc, bt.d[mine.di].q) : 0.0f;
          }
        }
      }
      return shfl_ref(mine, (int)(k & 31u));
    };
    uint32_t j_id = blockIdx.x;
    for (int s = 0; s < nst; ++s) {
      const uint32_t id = blockIdx.x + (uint32_t)s * gridDim.x;
      Stage<T> st = stage_at<T>(smem_raw, se, s);
      if (id < total) {
        const TileRef r = ref_of((uint32_t)s);
        produce<T, V>(bt, r, st, &refs[s], &full[s], lane);
      }
    }
    uint32_t done_phase = 0;
    int s = 0;
    for (uint32_t k = 0; j_id < total; j_id += gridDim.x, ++k) {
      // locate the refill tile while the consumers still work on this one
      const uint32_t nid = j_id + (uint32_t)nst * gridDim.x;
      TileRef nr;
      if (nid < total) nr = ref_of(k + (uint32_t)nst);
      const uint32_t par = (done_phase >> s) & 1u;
      mbar_wait(&done[s], par);
      done_phase ^= 1u << s;
      Stage<T> st = stage_at<T>(smem_raw, se, s);
      const TileRef cur = refs[s];
      const BwdDesc& d = bt.d[cur.di];
      if constexpr ((V & kProbeNoLoads) == 0) {
        store_dx<T>(d, cur, st, lane);
        if (lane == 0) bulk_wait_read_all();  // the store has read the stage
      }
      __syncwarp();
      if (nid < total) produce<T, V>(bt, nr, st, &refs[s], &full[s], lane, true);
      if constexpr ((V & kL2Pre) != 0) {
        // the tile one refill further ahead: into L2 now, so its TMA load
        // (issued when this stage frees up again) hits L2 instead of DRAM
        const uint32_t pid = nid + gridDim.x;
        if (pid < total) {
          const TileRef pr = ref_of(k + (uint32_t)nst + 1u);
          if (lane == 0 && pr.w1 > pr.w0) {
            const BwdDesc& pd = bt.d[pr.di];
            bulk_prefetch_l2(static_cast<const char*>(pd.x) + pr.w0, (uint32_t)(pr.w1 - pr.w0));
            bulk_prefetch_l2(static_cast<const char*>(pd.up) + pr.w0, (uint32_t)(pr.w1 - pr.w0));
          }
        }
      }
      // the tile's sums are read after the refill was issued (the next use
      // of this stage writes the other buffer)
      if constexpr ((V & kWarpPart) == 0) {
        const double part = lane_subtree(d, red[2 * s + par], lane);
        tile_sum(d, cur, part);
      } else {
        double w = lane < CW ? red[2 * s + par][lane] : 0.0;
#pragma unroll
        for (int o = 1; o < CW; o <<= 1) w = __dadd_rn(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (lane == 0) d.partials[((uint64_t)cur.seg << d.part_log) + cur.t] = w;
      }
      s = s + 1 == nst ? 0 : s + 1;
    }
    if (lane == 0) bulk_wait_all();
    return;
  }

  // ------------------------------- consumer warps ----------------------
  uint32_t full_phase = 0;
  GroupCache gc;
  PairCache pc;
  int s = 0;
  for (uint32_t tile_id = blockIdx.x; tile_id < total; tile_id += gridDim.x) {
    const uint32_t par = (full_phase >> s) & 1u;
    mbar_wait(&full[s], par);
    full_phase ^= 1u << s;
    Stage<T> st = stage_at<T>(smem_raw, se, s);
    const TileRef cur = refs[s];
    const BwdDesc& d = bt.d[cur.di];

    DivCtx dc;
    dc.s = pin(cur.s);
    dc.y = pin(cur.y);
    dc.ylo = (V & kDDiv) ? pin(recip_lo(cur.s, cur.y)) : 0.0;
    dc.usable = cur.s >= 0x1p-100 && cur.s <= 0x1p100;
    const double q = pin(d.q);
    double v;
    if constexpr ((V & kQuad) != 0) {
      int plo, pm;
      pc.get(cur.m, (int)d.g, tid, plo, pm);
      T* sx = st.x + cur.off + plo;
      const T* su = st.up + cur.off + plo;
      constexpr int kM = math_of<V>();
      if constexpr ((V & kHalfF32) != 0 && sizeof(T) == 2) {
        const HalfCtx hc = make_half_ctx(dc, q, cur.hthr);
        v = (d.dx != nullptr) ? quad_sum_h32<true>(sx, su, pm, dc, q, hc) : quad_sum_h32<false>(sx, su, pm, dc, q, hc);
      } else {
        v = (V & kProbeNoCompute) ? 0.0
          : (d.dx != nullptr && !(V & kProbeNoLoads)) ? quad_sum<T, true, kM>(sx, su, pm, dc, q)
                                                       : quad_sum<T, false, kM>(sx, su, pm, dc, q);
      }
    } else {
      int glo, glen;
      gc.get(cur.m, (int)d.g, tid, glo, glen);
      T* sx = st.x + cur.off + glo;
      const T* su = st.up + cur.off + glo;
      constexpr int kM = math_of<V>();
      v = (V & kProbeNoCompute) ? 0.0
        : (d.dx != nullptr && !(V & kProbeNoLoads)) ? group_sum_any<T, true, kM>(sx, su, glen, dc, q)
                                                     : group_sum_any<T, false, kM>(sx, su, glen, dc, q);
    }
    if constexpr ((V & kWarpPart) != 0) {
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) red[2 * s + par][warp] = v;  // the producer combines the 8 warp sums
    } else {
      red[2 * s + par][tid] = v;  // the producer runs the tile's tree reduction
    }
    // d_input was written into the stage with generic stores and leaves it
    // through a TMA bulk store (async proxy): every writing thread orders
    // its stores before the handoff (the TMA-store pattern). Measured:
    // consumer warps copying their own ranges out instead (coalesced
    // stores, no producer store) cost 19 M more instructions per frame and
    // 14 us.
    fence_proxy_async_smem();
    __syncwarp();     // the warp's d_input and group sums are written
    if (lane == 0) mbar_arrive(&done[s]);
    s = s + 1 == nst ? 0 : s + 1;
  }
}

// ---------------------------------------------------------------------
// CTA-uniform main pass (kCU, QFB_BWD_IMPL=tile...u): the forward chain
// kernel's pipeline shape for the backward's tree tiles. 8 warps, no
// producer warp: warp 0 locates tiles (32 at a time) and its lane 0 issues
// the TMA refill of the stage the previous iteration freed, NS-1 tiles
// ahead; every warp computes its 32 leaf groups, writes d_input into the
// stage and its warp sum; ONE CTA barrier per tile; then warp 0 combines
// the 8 warp sums into the tile partial and sends d_input out (ragged ends
// by lanes, the aligned interior by one bulk store). A stage is refilled
// one iteration later, after that store has read it.
// ---------------------------------------------------------------------
constexpr int kCU = 16384;
constexpr int kCuThreadStore = 32768;  // probe: d_input copied out by all threads (no TMA store)

template <typename T, int V>
__global__ void __launch_bounds__(kBwdThreads, 3) bwd_cu_kernel(const __grid_constant__ BwdBatch bt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ TileRef refs[kMaxStages];
  __shared__ double wsum[kMaxStages][kConsumerWarps];
  const int nst = bt.nstages;
  const uint32_t se = bt.stage_elems;
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t total = bt.tile_begin[bt.n];
  pdl_wait();
  if (blockIdx.x >= total) return;
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    pdl_trigger();
  }
  __syncthreads();

  // warp 0's tile locator (as the warp-specialized producer's)
  TileRef mine;
  uint32_t batch = 0xffffffffu;
  auto ref_of = [&](uint32_t k) -> TileRef {
    const uint32_t b = k >> 5;
    if (b != batch) {
      batch = b;
      const uint32_t id = blockIdx.x + ((b << 5) + (uint32_t)lane) * gridDim.x;
      if (id < total) mine = locate_full<T>(bt, id);
    }
    return shfl_ref(mine, (int)(k & 31u));
  };
  if (warp == 0) {
    for (int s = 0; s < nst - 1; ++s) {
      const uint32_t id = blockIdx.x + (uint32_t)s * gridDim.x;
      if (id < total) {
        Stage<T> st = stage_at<T>(smem_raw, se, s);
        produce<T, V>(bt, ref_of((uint32_t)s), st, &refs[s], &full[s], lane);
      }
    }
  }
  GroupCache gc;
  uint32_t full_phase = 0;
  int s = 0;
  for (uint32_t k = 0, tile_id = blockIdx.x; tile_id < total; tile_id += gridDim.x, ++k) {
    if (warp == 0) {
      // refill the stage freed by the previous iteration with tile k+nst-1
      const uint32_t nid = tile_id + (uint32_t)(nst - 1) * gridDim.x;
      if (nid < total) {
        const int rs = (s + nst - 1) % nst;
        const TileRef nr = ref_of(k + (uint32_t)nst - 1u);
        if (lane == 0) bulk_wait_read_all();  // that stage's d_input store has read it
        __syncwarp();
        Stage<T> st = stage_at<T>(smem_raw, se, rs);
        produce<T, V>(bt, nr, st, &refs[rs], &full[rs], lane, true);
      }
    }
    const uint32_t par = (full_phase >> s) & 1u;
    mbar_wait(&full[s], par);
    full_phase ^= 1u << s;
    Stage<T> st = stage_at<T>(smem_raw, se, s);
    const TileRef cur = refs[s];
    const BwdDesc& d = bt.d[cur.di];
    double v = 0.0;
    if constexpr ((V & kProbeNoCompute) == 0) {
      DivCtx dc;
      dc.s = pin(cur.s);
      dc.y = pin(cur.y);
      dc.ylo = (V & kDDiv) ? pin(recip_lo(cur.s, cur.y)) : 0.0;
      dc.usable = cur.s >= 0x1p-100 && cur.s <= 0x1p100;
      const double q = pin(d.q);
      int glo, glen;
      gc.get(cur.m, (int)d.g, tid, glo, glen);
      T* sx = st.x + cur.off + glo;
      const T* su = st.up + cur.off + glo;
      constexpr int kM = math_of<V>();
      v = d.dx != nullptr ? group_sum_any<T, true, kM>(sx, su, glen, dc, q)
                          : group_sum_any<T, false, kM>(sx, su, glen, dc, q);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    if (lane == 0) wsum[s][warp] = v;
    fence_proxy_async_smem();  // d_input leaves through the async proxy
    __syncthreads();           // the tile's d_input and warp sums are in shared memory
    if constexpr ((V & kCuThreadStore) != 0) {
      // probe: every thread copies d_input out with 16-byte stores, then a
      // second barrier frees the stage (no TMA store)
      if (d.dx != nullptr && d.vec) {
        const uint64_t b0 = cur.A * sizeof(T), b1 = (cur.A + (uint64_t)cur.m) * sizeof(T);
        const uint64_t i0 = (b0 + 15) & ~uint64_t(15), i1 = b1 & ~uint64_t(15);
        for (uint64_t o = i0 + (uint64_t)tid * 16; o < i1; o += 16 * kBwdThreads)
          *reinterpret_cast<uint4*>(static_cast<char*>(d.dx) + o) =
              *reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(st.x) + (o - cur.w0));
        if (warp == 0) {
          const int head = (int)(((i0 > b1 ? b1 : i0) - b0) / sizeof(T));
          const int tail0 = i1 > i0 ? (int)((i1 - b0) / sizeof(T)) : head;
          for (int e = lane; e < head; e += 32) static_cast<T*>(d.dx)[cur.A + e] = st.x[cur.off + e];
          for (int e = tail0 + lane; e < cur.m; e += 32) static_cast<T*>(d.dx)[cur.A + e] = st.x[cur.off + e];
        }
      } else if (warp == 0) {
        store_dx<T>(d, cur, st, lane);
      }
      if (warp == 0) {
        double w = lane < kConsumerWarps ? wsum[s][lane] : 0.0;
#pragma unroll
        for (int o = 1; o < kConsumerWarps; o <<= 1) w = __dadd_rn(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (lane == 0) d.partials[((uint64_t)cur.seg << d.part_log) + cur.t] = w;
      }
      __syncthreads();
    } else if (warp == 0) {
      double w = lane < kConsumerWarps ? wsum[s][lane] : 0.0;
#pragma unroll
      for (int o = 1; o < kConsumerWarps; o <<= 1) w = __dadd_rn(w, __shfl_xor_sync(0xffffffffu, w, o));
      if (lane == 0) d.partials[((uint64_t)cur.seg << d.part_log) + cur.t] = w;
      store_dx<T>(d, cur, st, lane);
    }
    s = s + 1 == nst ? 0 : s + 1;
  }
  if (warp == 0 && lane == 0) bulk_wait_all();
}

// Finisher: one warp per (descriptor, channel). Each row's 2^part_log tile
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
  const uint32_t tps = 1u << d.part_log;
  const uint32_t lanes = tps < 32u ? tps : 32u;
  const uint32_t per = tps / lanes;
  pdl_trigger();
  pdl_wait();  // see bwd_finish_reg_kernel
  const double chain = d.chain[c];
  double acc = 0.0;
  for (uint32_t o = 0; o < d.outer; ++o) {
    const double* p = d.partials + (((uint64_t)o * d.chans + c) << d.part_log);
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
    // accumulate == 0: ((r0 + r1) + ...); 1: ((d_log_s + r0) + r1) + ...;
    // QFB_BWD_ROWS: every row's r stored on its own
    if (d.accumulate == 2) {
      if (lane == 0) d.d_log_s[(uint64_t)o * d.row_stride + c] = r;
    } else if (o == 0) {
      acc = d.accumulate ? __dadd_rn(d.d_log_s[c], r) : r;
    } else {
      acc = __dadd_rn(acc, r);
    }
  }
  if (lane == 0 && d.accumulate != 2) d.d_log_s[c] = acc;
  (void)warp_base_mul;
}

// Register finisher for rows of <= 256 tiles (every DPVO shape): no shared
// memory (so 32 warps per SM hide the partials' load latency), each lane's
// `per` consecutive partials folded as a perfect subtree in registers, and
// four rows (frames) of a channel loaded before they are folded in row order.
// Same tree and fold order as bwd_finish_kernel.
template <int PER>
__device__ __forceinline__ double lane_slice(const double* p, int lane) {
  double a[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) a[k] = p[lane * PER + k];
#pragma unroll
  for (int w = PER; w > 1; w >>= 1)
#pragma unroll
    for (int k = 0; k < w / 2; ++k) a[k] = __dadd_rn(a[2 * k], a[2 * k + 1]);
  return a[0];
}

// per = 8 * M consecutive partials: M perfect subtrees of 8, then the
// perfect tree over their M sums (perfect trees compose).
template <int M>
__device__ __forceinline__ double lane_slice_wide(const double* p, int lane) {
  double a[M];
  const double* base = p + (size_t)lane * 8 * M;
#pragma unroll
  for (int g = 0; g < M; ++g) a[g] = lane_slice<8>(base + 8 * g, 0);
#pragma unroll
  for (int w = M; w > 1; w >>= 1)
#pragma unroll
    for (int k = 0; k < w / 2; ++k) a[k] = __dadd_rn(a[2 * k], a[2 * k + 1]);
  return a[0];
}

__device__ __forceinline__ double lane_slice_any(const double* p, int lane, uint32_t per) {
  switch (per) {
    case 1: return p[lane];
    case 2: return lane_slice<2>(p, lane);
    case 4: return lane_slice<4>(p, lane);
    case 8: return lane_slice<8>(p, lane);
    case 16: return lane_slice_wide<2>(p, lane);
    case 32: return lane_slice_wide<4>(p, lane);
    default: return lane_slice_wide<8>(p, lane);
  }
}

constexpr uint32_t kFinRegMaxTiles = 2048;  // per <= 64
constexpr int kFinRows = 4;

// early_chain: the chain factors were written before the main pass started
// (the main pass is not itself a programmatic dependent), so they may be
// read before griddepcontrol.wait, overlapping one load latency with the
// main pass's tail.
template <int WPB>
__global__ void __launch_bounds__(32 * WPB) bwd_finish_reg_kernel(const __grid_constant__ BwdBatch bt, uint32_t early_chain) {
  // WPB independent warps per CTA (fewer CTAs to launch); warp-local work only
  uint32_t w = blockIdx.x * WPB + (threadIdx.x >> 5);
  int di = 0;
  while (di < bt.n && w >= bt.d[di].chans) {
    w -= bt.d[di].chans;
    ++di;
  }
  if (di >= bt.n) return;
  const BwdDesc& d = bt.d[di];
  const uint32_t c = w;
  const int lane = threadIdx.x & 31;
  const uint32_t tps = 1u << d.part_log;
  const uint32_t lanes = tps < 32u ? tps : 32u;
  const uint32_t per = tps / lanes;
  const bool on = (uint32_t)lane < lanes;
  // prologue above overlaps the main pass's tail; d_log_s and the partials
  // are read only after it has completed
  pdl_trigger();
  double chain = early_chain ? d.chain[c] : 0.0;
  pdl_wait();
  if (!early_chain) chain = d.chain[c];
  const bool rows = d.accumulate == 2;
  double acc = d.accumulate == 1 ? d.d_log_s[c] : 0.0;
  for (uint32_t o = 0; o < d.outer; o += kFinRows) {
    double v[kFinRows];
#pragma unroll
    for (int j = 0; j < kFinRows; ++j) {
      v[j] = 0.0;
      if (on && o + j < d.outer)
        v[j] = lane_slice_any(d.partials + (((uint64_t)(o + j) * d.chans + c) << d.part_log), lane, per);
    }
#pragma unroll
    for (int j = 0; j < kFinRows; ++j) {
      for (uint32_t off = 1; off < lanes; off <<= 1)
        v[j] = __dadd_rn(v[j], __shfl_xor_sync(0xffffffffu, v[j], off));
      if (o + j < d.outer) {
        const double r = __dmul_rn(v[j], chain);
        // accumulate == 0: ((r0 + r1) + ...); 1: ((d_log_s + r0) + r1) + ...;
        // QFB_BWD_ROWS: every row's r stored on its own
        if (rows) {
          if (lane == 0) d.d_log_s[(uint64_t)(o + j) * d.row_stride + c] = r;
        } else {
          acc = (o + j == 0 && d.accumulate == 0) ? r : __dadd_rn(acc, r);
        }
      }
    }
  }
  if (lane == 0 && !rows) d.d_log_s[c] = acc;
}

// =====================================================================
// Streaming backward (sbwd_kernel). The memory-pipeline probe
// (tools/pipe_probe.cu, profiles/r02_pipe_probe.txt) moves this traffic
// shape (read x and up, write d_input) at 0.95-1.01 of measured HBM with
// ANY ring structure (register loads, TMA + CTA barrier, warp-specialized
// TMA with register or bulk stores), so the tile kernel's deficit was its
// per-tile work, not the pipeline. Here the pipeline carries no tree logic:
//   chunk = kSbChunk consecutive elements of one row (16-byte aligned: rows
//           of eligible tensors are 16-byte multiples), staged by TMA
//           together with the overhang of its last tree block and a
//           96-byte metadata record (its block starts, built once per row
//           shape by the host);
//   block = a node at depth D - 4 of the row's pairwise tree (16 leaf
//           groups, <= 256 elements); a chunk OWNS the blocks that start
//           inside it and folds them completely (their overhang is in its
//           window); d_input is stored for the chunk's own elements only.
// Warp roles (no CTA barrier after the prologue): one producer warp issues
// the stage refills (metadata prefetched one issue ahead); consumer warp w
// takes the chunk's blocks 2w and 2w+1 (32 leaf groups): phase 1 computes
// every element of its range lane-strided (4 independent elements per lane
// in flight: exact double quotient, term d_ds * up, d_input stored
// coalesced from registers) into a per-warp term buffer, releases the
// stage (one arrive per warp on `empty`), then phase 2: each half-warp
// folds one block — lane l folds leaf group l in the reference order (two
// <= 8 folds) and a 4-level xor butterfly forms the block's perfect-tree
// sum. The head of the chunk (elements before its first block, owned by
// the previous chunk's last block) gets its d_input from the first warp
// without blocks. Block partials feed the same finisher (part_log = D - 4).
// =====================================================================
constexpr int kSbConsumers = kSbThreads / 32;       // 8
constexpr int kSbCtaThreads = kSbThreads + 32;      // + producer warp
constexpr int kSbWarpTerms = kSbWarpBlocks * kSbMaxBlk;  // terms of a warp's blocks

struct SbRef {
  uint32_t di, row, c0, c1;  // descriptor, row (o * chans + c), chunk [c0, c1) of the row
  double s, y;               // scale and RN(1/s)
};

__device__ __forceinline__ void sb_decode(const BwdBatch& bt, uint32_t chunk, int& di, uint32_t& row,
                                          uint32_t& k) {
  int lo = 0, hi = bt.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bt.tile_begin[mid] <= chunk) lo = mid;
    else hi = mid - 1;
  }
  di = lo;
  const BwdDesc& d = bt.d[lo];
  const uint32_t local = chunk - bt.tile_begin[lo];
  row = fdiv(local, d.sb_nch_div);
  k = local - row * d.sb_nch;
}

// Fold of one leaf group's terms in the reference order (tensor.hpp:100-109
// below the block: n <= 8 -> left fold from 0.0, else fold(first n/2) +
// fold(rest)). Groups here hold 8..16 terms.
__device__ __forceinline__ double sb_group_fold(const double* t, int len) {
  if (len <= 8) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < len) acc = __dadd_rn(acc, t[k]);
    return acc;
  }
  const int h = len >> 1;
  const double* r = t + h;
  double al = 0.0, ar = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (k < h) al = __dadd_rn(al, t[k]);
    if (k < len - h) ar = __dadd_rn(ar, r[k]);
  }
  return __dadd_rn(al, ar);
}

// One element: term (double) and d_input bits, exact reference semantics.
template <typename T>
__device__ __forceinline__ double sb_elem(T xe, T ue, const DivCtx& dc, double q, T& dxo) {
  if (dc.usable) {
    double t;
    if constexpr (sizeof(T) == 4) {
      float dd;
      t = fast_term(xe, ue, dc, q, dd);
      dxo = dd;
    } else {
      t = fast_term_h(xe, ue, dc, q, &dxo);
    }
    const float uf = to_f<T>(ue);
    if (__builtin_expect((__float_as_uint(uf) & 0x7f800000u) == 0x7f800000u, 0))
      dxo = from_f<T>(masked_upstream(grad_term(to_f<T>(xe), dc.s, q).mask, uf));
    return t;
  }
  const double2 t2 = slow_elem(to_f<T>(xe), to_f<T>(ue), dc.s, q);
  dxo = from_f<T>((float)t2.y);
  return t2.x;
}

// Phase 1 of one warp over the row elements [lo, hi) (window-relative
// views sx / su): lane-strided (consecutive lanes, consecutive elements:
// conflict-free shared reads, coalesced d_input stores), 4 independent
// elements per lane in flight in the unchecked main loop, then 32-element
// steps. Terms (kTerms) go to the warp's buffer at [i - lo]; d_input is
// stored for i < c1 (kDxCheck: only the warp whose range crosses c1 tests
// it). kUsable is the chunk-uniform scale test of the fast quotient.
template <typename T, bool kUsable>
__device__ __forceinline__ double sb_term(T xe, T ue, const DivCtx& dc, double q, T& dv, uint32_t& bad) {
  if constexpr (kUsable) {
    bad |= (__float_as_uint(to_f<T>(ue)) & 0x7f800000u) == 0x7f800000u ? 1u : 0u;
    if constexpr (sizeof(T) == 4) {
      float dd;
      const double t = fast_term(xe, ue, dc, q, dd);
      dv = dd;
      return t;
    } else {
      return fast_term_h(xe, ue, dc, q, &dv);
    }
  } else {
    const double2 t2 = slow_elem(to_f<T>(xe), to_f<T>(ue), dc.s, q);
    dv = from_f<T>((float)t2.y);
    return t2.x;
  }
}

template <typename T>
__device__ __noinline__ T sb_fix_dx(T xe, T ue, const DivCtx& dc, double q, T dv) {
  // non-finite upstream: the reference's d_input rules (rare)
  const float uf = to_f<T>(ue);
  if ((__float_as_uint(uf) & 0x7f800000u) == 0x7f800000u)
    return from_f<T>(masked_upstream(grad_term(to_f<T>(xe), dc.s, q).mask, uf));
  return dv;
}

template <typename T, bool kUsable, bool kTerms, bool kDxCheck>
__device__ __forceinline__ void sb_sweep(const T* sx, const T* su, uint32_t lo, uint32_t hi, uint32_t c1,
                                         const DivCtx& dc, double q, double* terms, T* dxrow) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t n = hi - lo;
  const uint32_t nd = c1 > lo ? c1 - lo : 0u;  // d_input for relative index < nd
  const T* px = sx + lo;
  const T* pu = su + lo;
  T* pd = dxrow ? dxrow + lo : nullptr;
  uint32_t i = lane;
  for (; i + 96u < n; i += 128u) {
    double tv[4];
    T dv[4], xe[4], ue[4];
    uint32_t bad = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      xe[k] = px[i + 32u * k];
      ue[k] = pu[i + 32u * k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) tv[k] = sb_term<T, kUsable>(xe[k], ue[k], dc, q, dv[k], bad);
    if (kUsable && __builtin_expect(bad != 0, 0)) {
#pragma unroll
      for (int k = 0; k < 4; ++k) dv[k] = sb_fix_dx<T>(xe[k], ue[k], dc, q, dv[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (kTerms) terms[i + 32u * k] = tv[k];
      if (pd && (!kDxCheck || i + 32u * k < nd)) pd[i + 32u * k] = dv[k];
    }
  }
  for (; i < n; i += 32u) {
    T dv;
    uint32_t bad = 0;
    const T xe = px[i], ue = pu[i];
    const double tv = sb_term<T, kUsable>(xe, ue, dc, q, dv, bad);
    if (kUsable && __builtin_expect(bad != 0, 0)) dv = sb_fix_dx<T>(xe, ue, dc, q, dv);
    if (kTerms) terms[i] = tv;
    if (pd && (!kDxCheck || i < nd)) pd[i] = dv;
  }
}

// Fold of a leaf group of 9 or 10 terms (every group of the DPVO rows:
// n / 2^D = 9.375) in the reference order: fold(first 4 or 5) + fold(5).
__device__ __forceinline__ double sb_group_fold_9_10(const double* t, int len) {
  const int h = len >> 1;  // 4 or 5
  const double* r = t + h;
  double al = __dadd_rn(0.0, t[0]), ar = __dadd_rn(0.0, r[0]);
#pragma unroll
  for (int k = 1; k < 4; ++k) {
    al = __dadd_rn(al, t[k]);
    ar = __dadd_rn(ar, r[k]);
  }
  if (h == 5) al = __dadd_rn(al, t[4]);
  ar = __dadd_rn(ar, r[4]);
  return __dadd_rn(al, ar);
}

template <typename T, int NS>
__global__ void __launch_bounds__(kSbCtaThreads, 3) sbwd_kernel(const __grid_constant__ BwdBatch bt) {
  constexpr uint32_t kWinBytes = kSbWin * sizeof(T);
  constexpr uint32_t kStageBytes = 2 * kWinBytes + kSbMetaWords * 4;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[NS];
  __shared__ __align__(8) uint64_t empty[NS];
  __shared__ SbRef refs[NS];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const uint32_t total = bt.tile_begin[bt.n];
  pdl_wait();
  if (blockIdx.x >= total) return;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kSbConsumers);
    }
    fence_mbar_init();
    pdl_trigger();
  }
  __syncthreads();  // the only CTA barrier: barrier init

  if (warp == kSbConsumers) {
    // ------------------------------------------------ producer warp ----
    if (lane != 0) return;
    uint32_t nx_chunk = 0, nx_row = 0, nx_k = 0, nx_le = 0;
    int nx_di = 0;
    double nx_s = 1.0;
    auto prefetch = [&](uint32_t chunk) {
      nx_chunk = chunk;
      if (chunk >= total) return;
      sb_decode(bt, chunk, nx_di, nx_row, nx_k);
      const BwdDesc& d = bt.d[nx_di];
      nx_le = __ldg(d.sb_meta + (size_t)nx_k * kSbMetaWords + 2);
      nx_s = __ldg(d.s64 + (nx_row % d.chans));
    };
    auto issue = [&](int stage) {
      const BwdDesc& d = bt.d[nx_di];
      const uint32_t n = (uint32_t)d.inner;
      const uint32_t c0 = nx_k * (uint32_t)kSbChunk;
      const uint32_t c1 = min(c0 + (uint32_t)kSbChunk, n);
      constexpr uint32_t V = 16 / sizeof(T);
      uint32_t end = max(c1, nx_le);
      end = min((end + V - 1) & ~(V - 1), n);
      SbRef r;
      r.di = (uint32_t)nx_di;
      r.row = nx_row;
      r.c0 = c0;
      r.c1 = c1;
      r.s = nx_s;
      r.y = __drcp_rn(nx_s);
      refs[stage] = r;
      const uint32_t bytes = (end - c0) * (uint32_t)sizeof(T);
      unsigned char* st = smem_raw + (size_t)stage * kStageBytes;
      const uint64_t off = ((uint64_t)nx_row * d.inner + c0) * sizeof(T);
      mbar_arrive_expect_tx(&full[stage], 2 * bytes + kSbMetaWords * 4);
      bulk_g2s(st, static_cast<const char*>(d.x) + off, bytes, &full[stage]);
      bulk_g2s(st + kWinBytes, static_cast<const char*>(d.up) + off, bytes, &full[stage]);
      bulk_g2s(st + 2 * kWinBytes, d.sb_meta + (size_t)nx_k * kSbMetaWords, kSbMetaWords * 4, &full[stage]);
    };
    prefetch(blockIdx.x);
    uint32_t phase = 0;
    int s = 0;
    for (uint32_t it = 0; nx_chunk < total; ++it) {
      if (it >= (uint32_t)NS) {
        mbar_wait_sleep(&empty[s], (phase >> s) & 1u);  // all consumer warps are done reading stage s
        phase ^= 1u << s;
      }
      issue(s);
      prefetch(nx_chunk + gridDim.x);
      s = s + 1 == NS ? 0 : s + 1;
    }
    return;
  }

  // ------------------------------------------------- consumer warps ----
  double* terms = reinterpret_cast<double*>(smem_raw + (size_t)NS * kStageBytes) + (size_t)warp * kSbWarpTerms;
  uint32_t phase = 0;
  int s = 0;
  for (uint32_t chunk = blockIdx.x; chunk < total; chunk += gridDim.x) {
    mbar_wait_sleep(&full[s], (phase >> s) & 1u);
    phase ^= 1u << s;
    const SbRef r = refs[s];
    const BwdDesc& d = bt.d[r.di];
    const unsigned char* st = smem_raw + (size_t)s * kStageBytes;
    const uint32_t* meta = reinterpret_cast<const uint32_t*>(st + 2 * kWinBytes);
    // window-relative element views of the staged x and upstream
    const T* sx = reinterpret_cast<const T*>(st) - r.c0;
    const T* su = reinterpret_cast<const T*>(st + kWinBytes) - r.c0;
    DivCtx dc;
    dc.s = r.s;
    dc.y = r.y;
    dc.usable = r.s >= 0x1p-100 && r.s <= 0x1p100;
    const double q = d.q;
    T* dxrow = d.dx ? static_cast<T*>(d.dx) + (uint64_t)r.row * d.inner : nullptr;
    const uint32_t nblk = meta[1];
    const uint32_t b0 = (uint32_t)kSbWarpBlocks * (uint32_t)warp;  // this warp's blocks (chunk-relative)
    const uint32_t nb = nblk > b0 ? min(nblk - b0, (uint32_t)kSbWarpBlocks) : 0u;
    const uint32_t a = nb ? meta[4 + b0] : 0u;  // this warp's range [a, e) of the row
    const uint32_t e = nb ? meta[4 + b0 + nb] : 0u;
    const uint32_t blo0 = 0u, bm0 = nb ? meta[5 + b0] - a : 0u;
    const uint32_t blo1 = bm0, bm1 = nb > 1 ? e - meta[5 + b0] : 0u;
    const uint32_t jb = meta[0] + b0;
    // the chunk head [c0, first block) belongs to the previous chunk's last
    // block: its d_input comes from the first warp without blocks (warp 7
    // when all have blocks)
    const bool head =
        (uint32_t)warp == min((nblk + kSbWarpBlocks - 1u) / kSbWarpBlocks, (uint32_t)kSbConsumers - 1u);
    const uint32_t head_end = nblk ? meta[4] : r.c1;
    // ---- phase 1: this warp's elements, lane-strided, 4 in flight per lane
    if (dc.usable) {
      if (nb) {
        if (e <= r.c1) sb_sweep<T, true, true, false>(sx, su, a, e, r.c1, dc, q, terms, dxrow);
        else sb_sweep<T, true, true, true>(sx, su, a, e, r.c1, dc, q, terms, dxrow);
      }
      if (head) sb_sweep<T, true, false, false>(sx, su, r.c0, head_end, r.c1, dc, q, terms, dxrow);
    } else {
      if (nb) sb_sweep<T, false, true, true>(sx, su, a, e, r.c1, dc, q, terms, dxrow);
      if (head) sb_sweep<T, false, false, false>(sx, su, r.c0, head_end, r.c1, dc, q, terms, dxrow);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // stage s no longer read by this warp
    // ---- phase 2: one half-warp per block, from this warp's terms
    const int h = lane >> 4;
    const int l16 = lane & 15;
    double v = 0.0;
    const bool active = (uint32_t)h < nb;
    if (active) {
      uint32_t gl = 0, gm = h ? bm1 : bm0;
      descend<uint32_t>(gl, gm, (uint32_t)l16, kSbBlockLog);
      const double* tg = terms + (h ? blo1 : blo0) + gl;
      v = (gm == 9 || gm == 10) ? sb_group_fold_9_10(tg, (int)gm) : sb_group_fold(tg, (int)gm);
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (active && l16 == 0) d.partials[((uint64_t)r.row << d.part_log) + jb + h] = v;
    __syncwarp();  // terms read before the next chunk overwrites them
    s = s + 1 == NS ? 0 : s + 1;
  }
}

}  // namespace

// Ring budget per CTA (bytes) and stage cap; QFB_BWD_RING_KB /
// QFB_BWD_STAGES override them for tuning sweeps.
static size_t ring_budget() {
  static const size_t b = [] {
    const char* e = getenv("QFB_BWD_RING_KB");
    const long kb = e ? atol(e) : 0;
    return kb > 0 ? (size_t)kb * 1024 : kRingBudget;
  }();
  return b;
}
static int stage_cap() {
  static const int c = [] {
    const char* e = getenv("QFB_BWD_STAGES");
    const int v = e ? atoi(e) : 0;
    return v >= 2 && v <= kMaxStages ? v : kMaxStages;
  }();
  return c;
}

void bwd_ring_size(int dtype, uint32_t max_tile, uint32_t* stage_elems, int32_t* nstages,
                   size_t* smem_bytes) {
  const size_t es = dtype == 0 ? 4 : 2;
  uint32_t se = max_tile + kWinPad;
  se = (se + 7u) & ~7u;  // 16-byte multiple for both element sizes
  const size_t stage = 2 * (size_t)se * es;
  int ns = (int)(ring_budget() / (stage + kRedBytes));
  if (ns > stage_cap()) ns = stage_cap();
  if (ns < 2) ns = 2;
  *stage_elems = se;
  *nstages = ns;
  *smem_bytes = (stage + kRedBytes) * (size_t)ns;
}

namespace {

// Kernel variant: 0 = production; the probes (QFB_BWD_VARIANT=8 / 16)
// isolate the memory pipeline and the arithmetic for roofline analysis.
static int variant() {
  static const int v = [] {
    const char* e = getenv("QFB_BWD_VARIANT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

// A kernel instance and its block size.
struct BwdFn {
  const void* fn;
  int threads;
};
template <typename T, int V>
BwdFn bwd_inst() {
  if constexpr ((V & kCU) != 0) return BwdFn{(const void*)bwd_cu_kernel<T, V>, kBwdThreads};
  return BwdFn{(const void*)bwd_kernel<T, V>, cta_threads<V>()};
}

// The production instance for a batch: the generic kernel when some row
// has short tiles, else the full-tile kernel with the batch's consumer
// layout. QFB_BWD_VARIANT (diagnostics) selects the probes: 8 memory
// pipeline only, 16 arithmetic only (on the generic kernel, or with
// kQuad | kMagicRint set: on the quad kernel).
template <typename T>
BwdFn kernel_ptr(int v, bool warp_part, uint32_t layout) {
  layout &= ~kBwdLayoutReverse;  // a runtime bit, not an instance
  constexpr int kQM = kWarpPart | kQuad | kMagicRint;
  switch (v) {
    case kProbeNoCompute: return bwd_inst<T, kProbeNoCompute>();
    case kProbeNoLoads: return bwd_inst<T, kProbeNoLoads>();
    case kQM | kProbeNoCompute: if (warp_part) return bwd_inst<T, kQM | kProbeNoCompute>(); break;
    case kWarpPart | kDDiv | kProbeNoCompute:  // the production structure's memory-only probe
      if (warp_part) return bwd_inst<T, kWarpPart | kDDiv | kProbeNoCompute>();
      break;
    case kWarpPart | kDDiv | kProbeNoLoads:  // ... and its arithmetic-only probe
      if (warp_part) return bwd_inst<T, kWarpPart | kDDiv | kProbeNoLoads>();
      break;
    case kQM | kProbeNoLoads: if (warp_part) return bwd_inst<T, kQM | kProbeNoLoads>(); break;
    default: break;
  }
  if (!warp_part) return bwd_inst<T, 0>();
  static const bool two_env = [] {
    const char* e = getenv("QFB_BWD_CTAS");
    return e && e[0] == '2';
  }();
  if constexpr (sizeof(T) == 2)
    // float32 terms: the quad layout (cheap arithmetic, the faster memory
    // pipeline of 4 consumer warps: 75 us vs 80 us with 8 warps x 1 group)
    if (layout & kBwdLayoutHalfF32) return bwd_inst<T, kWarpPart | kQuad | kDDiv | kHalfF32>();
  const bool two = two_env || (layout & kBwdLayoutTwoCtas) != 0;
  if (two && (layout & ~kBwdLayoutTwoCtas) == kBwdLayoutDD) return bwd_inst<T, kWarpPart | kDDiv | kTwoCtas>();
  if ((layout & ~kBwdLayoutPrefetch) == kBwdLayoutDD && (layout & kBwdLayoutPrefetch))
    return bwd_inst<T, kWarpPart | kDDiv | kL2Pre>();
  if (layout & kBwdLayoutCU) {
    switch (v) {
      case 9: return bwd_inst<T, kWarpPart | kDDiv | kCU | kProbeNoCompute>();
      case 10: return bwd_inst<T, kWarpPart | kDDiv | kCU | kProbeNoCompute | kCuThreadStore>();
      case 11: return bwd_inst<T, kWarpPart | kDDiv | kCU | kCuThreadStore>();
      default: return bwd_inst<T, kWarpPart | kDDiv | kCU>();
    }
  }
  // layout bits: kBwdLayoutMagic | kBwdLayoutQuad | kBwdLayoutDD
  switch (layout & 7u) {
    case 1: return bwd_inst<T, kWarpPart | kMagicRint>();
    case 2: return bwd_inst<T, kWarpPart | kQuad>();
    case 3: return bwd_inst<T, kWarpPart | kQuad | kMagicRint>();
    case 4: return bwd_inst<T, kWarpPart | kDDiv>();
    case 5: return bwd_inst<T, kWarpPart | kMagicRint | kDDiv>();
    case 6: return bwd_inst<T, kWarpPart | kQuad | kDDiv>();
    case 7: return bwd_inst<T, kWarpPart | kQuad | kMagicRint | kDDiv>();
    default: return two ? bwd_inst<T, kWarpPart | kTwoCtas>() : bwd_inst<T, kWarpPart>();
  }
}

BwdFn bwd_fn(int dtype, bool warp_part, uint32_t layout) {
  return dtype == 0 ? kernel_ptr<float>(variant(), warp_part, layout)
                    : kernel_ptr<__half>(variant(), warp_part, layout);
}

}  // namespace

cudaError_t bwd_occupancy(int dtype, int* blocks_per_sm) {
  uint32_t se;
  int32_t ns;
  size_t smem;
  bwd_ring_size(dtype, kBwdTileMax, &se, &ns, &smem);
  return bwd_occupancy_smem(dtype, smem, blocks_per_sm);
}

cudaError_t bwd_occupancy_smem(int dtype, size_t smem, int* blocks_per_sm, bool warp_part, uint32_t layout) {
  const BwdFn f = bwd_fn(dtype, warp_part, layout);
  cudaError_t e = cudaFuncSetAttribute(f.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f.fn, f.threads, smem);
}

cudaError_t launch_bwd(int dtype, const BwdBatch& b, int grid, cudaStream_t st, cudaEvent_t after_main,
                       cudaStream_t fin_stream, cudaEvent_t fork) {
  const uint32_t tiles = b.tile_begin[b.n];
  if (tiles == 0) return cudaSuccess;
  if ((uint32_t)grid > tiles) grid = (int)tiles;
  const size_t smem = (size_t)b.nstages * (2 * b.stage_elems * (dtype == 0 ? 4 : 2) + kRedBytes);
  void* args[] = {const_cast<BwdBatch*>(&b)};
  static const cudaError_t hints_set = [] {
    const char* e = getenv("QFB_L2_HINTS");
    if (!(e && e[0])) return cudaSuccess;
    const int mask = (int)strtol(e, nullptr, 0);
    return cudaMemcpyToSymbol(c_bwd_l2_hints, &mask, sizeof mask);
  }();
  if (hints_set != cudaSuccess) return hints_set;
  const BwdFn f = bwd_fn(dtype, b.warp_part != 0, b.layout);
  cudaFuncSetAttribute(f.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemMax);
  cudaError_t e = launch_main(f.fn, dim3(grid), dim3(f.threads), args, smem, st, kPdlBwd);
  if (e != cudaSuccess) return e;
  if (after_main) {  // profiling hook (QFB_OPT_MAIN_PASS_EVENT)
    e = cudaEventRecord(after_main, st);
    if (e != cudaSuccess) return e;
  }
  // QFB_DIAG_SKIP_FINISH=1: timing diagnostic only (d_log_s is NOT written)
  static const bool skip_fin = [] {
    const char* e = getenv("QFB_DIAG_SKIP_FINISH");
    return e && e[0] == '1';
  }();
  if (skip_fin) return cudaSuccess;
  if (fin_stream) {  // QFB_OPT_BWD_ASYNC_FINISH: the finisher on the side stream
    e = cudaEventRecord(fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(fin_stream, fork, 0);
    if (e != cudaSuccess) return e;
    return launch_bwd_finish(b, fin_stream);
  }
  return launch_bwd_finish(b, st);
}

namespace {
constexpr int kSbStagesF32 = 3, kSbStagesF16 = 3;
const void* sbwd_fn(int dtype, int stages) {
  if (dtype == 0) {
    if (stages == 2) return (const void*)sbwd_kernel<float, 2>;
    if (stages == 4) return (const void*)sbwd_kernel<float, 4>;
    return (const void*)sbwd_kernel<float, 3>;
  }
  if (stages == 2) return (const void*)sbwd_kernel<__half, 2>;
  if (stages == 4) return (const void*)sbwd_kernel<__half, 4>;
  return (const void*)sbwd_kernel<__half, 3>;
}
}  // namespace

size_t sbwd_smem(int dtype, int stages) {
  const size_t es = dtype == 0 ? 4 : 2;
  return (size_t)stages * (2 * kSbWin * es + kSbMetaWords * 4) +
         (size_t)kSbConsumers * kSbWarpTerms * sizeof(double);
}

cudaError_t sbwd_occupancy(int dtype, int stages, int* blocks_per_sm) {
  const void* f = sbwd_fn(dtype, stages);
  const size_t smem = sbwd_smem(dtype, stages);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, kSbCtaThreads, smem);
}

cudaError_t launch_sbwd(int dtype, int stages, const BwdBatch& b, int grid, cudaStream_t st) {
  const uint32_t chunks = b.tile_begin[b.n];
  if (chunks == 0) return cudaSuccess;
  if ((uint32_t)grid > chunks) grid = (int)chunks;
  void* args[] = {const_cast<BwdBatch*>(&b)};
  cudaError_t e = launch_main(sbwd_fn(dtype, stages), dim3(grid), dim3(kSbCtaThreads), args,
                              sbwd_smem(dtype, stages), st, kPdlBwd);
  if (e != cudaSuccess) return e;
  return launch_bwd_finish(b, st);
}

cudaError_t launch_bwd_finish(const BwdBatch& b, cudaStream_t st) {
  cudaError_t e;
  uint32_t warps = 0, max_tps = 0;
  for (int i = 0; i < b.n; ++i) {
    warps += b.d[i].chans;
    max_tps = std::max(max_tps, 1u << b.d[i].part_log);
  }
  static const bool force_smem = [] {
    const char* e = getenv("QFB_FIN_SMEM");
    return e && e[0] == '1';
  }();
  uint32_t zero = 0;
  void* fargs[] = {const_cast<BwdBatch*>(&b), &zero};
  uint32_t early = pdl_enabled(kPdlBwd) ? 0u : 1u;
  void* rargs[] = {const_cast<BwdBatch*>(&b), &early};
  // warps per finisher CTA (QFB_FIN_WARPS 1/4/8): 4 measured best in the
  // step (0.1346 -> 0.1335 ms: fewer CTAs to launch after the main pass)
  static const int wpb = [] {
    const char* e = getenv("QFB_FIN_WARPS");
    const int v = e ? atoi(e) : 4;
    return v == 1 || v == 8 ? v : 4;
  }();
  if (max_tps <= kFinRegMaxTiles && !force_smem) {
    const void* fn = wpb == 8 ? (const void*)bwd_finish_reg_kernel<8>
                   : wpb == 4 ? (const void*)bwd_finish_reg_kernel<4> : (const void*)bwd_finish_reg_kernel<1>;
    e = launch_main(fn, dim3((warps + wpb - 1) / wpb), dim3(32 * wpb), rargs, 0, st, kPdlFin);
  }
  else
    e = launch_main((const void*)bwd_finish_kernel, dim3(warps), dim3(32), fargs, 0, st, kPdlFin);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace qfb
