// qfb_fwd.cu — forward-side sm_100a kernels: fused fake-quant forward /
// quant->act->quant chains (one HBM pass over a table of quant points),
// int8 code emission, the per-operator ablation sweeps, device scale
// resolution and the counter-RNG synthetic generator.
//
// All of these are HBM-bound elementwise sweeps (SURVEY.md §8 d): 16-byte
// vectorized, coalesced loads (ld.global.nc.L1::no_allocate) and stores,
// kEwUnroll independent loads in flight per thread, a grid of
// (SM count x resident CTAs) persistent CTAs striding over 1024-unit chunks.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdlib.h>

#include "../../include/qfb_portable.h"
#include "qfb_device.cuh"
#include "qfb_kernels.h"

namespace qfb {

namespace {

__device__ __forceinline__ uint32_t channel_of(uint32_t unit, const FastDiv& inner_u,
                                               const FastDiv& chans) {
  if (chans.d == 1) return 0;
  const uint32_t row = fdiv(unit, inner_u);
  return row - fdiv(row, chans) * chans.d;
}

__device__ __forceinline__ float apply_act(float v, int act) {
  if (act == 1) return v > 0.0f ? v : 0.0f;  // relu, tensor.hpp:147-151
  if (act == 2) return qfb_p_gelu(v);
  return v;
}

// FQ of one unit (V elements sharing scale s): division shortcut with the
// reciprocal hoisted per unit when the scale is in the proven range.
template <int V>
__device__ __forceinline__ void fq_unit(const float* v, float s, float q, float* o) {
  if (fast_div_ok(s)) {
    const float y = __frcp_rn(s);
#pragma unroll
    for (int i = 0; i < V; ++i) o[i] = fq_value_fast(v[i], s, y, q);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) o[i] = fq_value(v[i], s, q);
  }
}

// int8 codes of one unit (quant.hpp:174-207: (int8)nearbyintf(clip(x/s)),
// NaN -> 0), with the same proven division shortcut as the FQ value: the
// clipped, rounded quotient is identical to rint(clip(IEEE x/s)).
template <int V>
__device__ __forceinline__ void code_unit(const float* v, float s, float y, bool fast, float q,
                                          uint32_t* c, bool finite = false) {
  if (finite) {  // screened unit: no overflow guard, no NaN
#pragma unroll
    for (int i = 0; i < V; ++i) c[i] = fq_code_bits_fast_finite(v[i], s, y, q);
    return;
  }
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (fast) {
      const float q0 = __fmul_rn(v[i], y);
      float z = __fmaf_rn(__fmaf_rn(-s, q0, v[i]), y, q0);
      z = fabsf(q0) < 0x1p100f ? z : q0;
      z = fminf(fmaxf(copysignf(z, v[i]), -q), q);
      // round-to-nearest-even into the low byte: 1.5*2^23 + z, |z| <= q
      const uint32_t b = __float_as_uint(__fadd_rn(z, 12582912.0f));
      c[i] = isnan(v[i]) ? 0u : b;
    } else {
      c[i] = (uint32_t)(uint8_t)fq_code(v[i], s, q);
    }
  }
}

// f32 unit screen: every |x| < thr = s * 2^100 (false for NaN and inf, and
// thr = 0 when the scale is outside the shortcut's range).
template <int V>
__device__ __forceinline__ bool screen_f32(const float* v, float thr) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < V; ++i) ok = ok && fabsf(v[i]) < thr;
  return ok;
}

// Store V codes (low bytes of c) at unit u of an int8 output (V bytes).
template <int V>
__device__ __forceinline__ void store_codes(void* y, uint32_t u, const uint32_t* c) {
  uint32_t w[V / 4];
#pragma unroll
  for (int k = 0; k < V / 4; ++k)
    w[k] = __byte_perm(__byte_perm(c[4 * k], c[4 * k + 1], 0x0040), __byte_perm(c[4 * k + 2], c[4 * k + 3], 0x0040),
                       0x5410);
  if constexpr (V == 4) reinterpret_cast<uint32_t*>(y)[u] = w[0];
  else reinterpret_cast<uint2*>(y)[u] = make_uint2(w[0], w[1]);
}

// Vector path: every unit is one 16-byte vector, all its elements share a
// channel (host guarantees inner % kPerVec == 0 and 16-byte alignment).
// kChain = false is the plain multi-output fake-quant forward (no b, no
// activation, no preact, no demotion): fewer live registers, more CTAs/SM.
template <typename T, bool kChain>
__device__ __forceinline__ void ew_vec(const EwDesc& d, uint32_t ubase, bool& nf) {
  constexpr int V = Elem<T>::kPerVec;
  const bool streaming = (d.flags & kEwStreaming) != 0;
  const bool half_out = (d.flags & kEwHalfGrid) != 0;
  uint4 ra[kEwUnroll];
  uint4 rb[kChain ? kEwUnroll : 1];
  const bool has_b = kChain && d.b != nullptr;
#pragma unroll
  for (int k = 0; k < kEwUnroll; ++k) {
    const uint32_t u = ubase + k * kEwThreads;
    if (u < d.nunits) {
      ra[k] = ld_nc_v4(static_cast<const uint4*>(d.a) + u);
      if constexpr (kChain) {
        if (has_b) rb[k] = ld_nc_v4(static_cast<const uint4*>(d.b) + u);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kEwUnroll; ++k) {
    const uint32_t u = ubase + k * kEwThreads;
    if (u >= d.nunits) break;
    const uint32_t ch = channel_of(u, d.inner_u, d.chans);
    float v[V];
    Elem<T>::unpack(ra[k], v);
    if constexpr (kChain) {
      if (has_b) {
        float w[V];
        Elem<T>::unpack(rb[k], w);
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = x86_add(v[i], w[i]);  // tensor.hpp:126-134
      }
      if (d.act != 0) {
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = apply_act(v[i], d.act);
      }
      if (d.flags & kEwDemoteIn) {
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = half_grid(v[i], v[i], nf);  // tensor.hpp:159-170
      }
      if (d.preact != nullptr) {
        st_v4(static_cast<uint4*>(d.preact) + u, Elem<T>::pack(v, v, false, nf), streaming);
      }
    }
    for (int j = 0; j < d.n_out; ++j) {
      const float s = __ldg(d.s[j] + ch);
      if (d.flags & kEwInt8Out) {
        uint32_t c[V];
        code_unit<V>(v, s, fast_div_ok(s) ? __frcp_rn(s) : 1.0f, fast_div_ok(s), d.q, c);
        store_codes<V>(d.y[j], u, c);
        continue;
      }
      float o[V];
      fq_unit<V>(v, s, d.q, o);
      st_v4(static_cast<uint4*>(d.y[j]) + u, Elem<T>::pack(o, v, half_out, nf), streaming);
    }
  }
}

// Scalar path (unaligned or inner % kPerVec != 0): unit == element.
template <typename T>
__device__ __forceinline__ void ew_scalar(const EwDesc& d, uint32_t ubase, bool& nf) {
  const bool has_b = d.b != nullptr;
  const bool half_out = (d.flags & kEwHalfGrid) != 0;
  const bool demote_in = (d.flags & kEwDemoteIn) != 0;
  float va[kEwUnroll], vb[kEwUnroll];
#pragma unroll
  for (int k = 0; k < kEwUnroll; ++k) {
    const uint32_t u = ubase + k * kEwThreads;
    if (u < d.nunits) {
      va[k] = Elem<T>::load1(d.a, u);
      vb[k] = has_b ? Elem<T>::load1(d.b, u) : 0.0f;
    }
  }
#pragma unroll
  for (int k = 0; k < kEwUnroll; ++k) {
    const uint32_t u = ubase + k * kEwThreads;
    if (u >= d.nunits) break;
    const uint32_t ch = channel_of(u, d.inner_u, d.chans);
    float v = va[k];
    if (has_b) v = x86_add(v, vb[k]);
    v = apply_act(v, d.act);
    if (demote_in) v = half_grid(v, v, nf);
    if (d.preact != nullptr) Elem<T>::store1(d.preact, u, v, v, false, nf);
    for (int j = 0; j < d.n_out; ++j) {
      if (d.flags & kEwInt8Out) {
        static_cast<int8_t*>(d.y[j])[u] = fq_code(v, __ldg(d.s[j] + ch), d.q);
        continue;
      }
      float o;
      fq_unit<1>(&v, __ldg(d.s[j] + ch), d.q, &o);
      Elem<T>::store1(d.y[j], u, o, v, half_out, nf);
    }
  }
}

template <typename T, bool kChain>
__global__ void __launch_bounds__(kEwThreads, kChain ? 3 : 4) ew_kernel(const __grid_constant__ EwBatch bt,
                                                        uint32_t* __restrict__ status) {
  bool nf = false;
  const uint32_t total = bt.chunk_begin[bt.n];
  for (uint32_t chunk = blockIdx.x; chunk < total; chunk += gridDim.x) {
    int lo = 0, hi = bt.n - 1;  // last descriptor with chunk_begin <= chunk
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (bt.chunk_begin[mid] <= chunk) lo = mid;
      else hi = mid - 1;
    }
    const EwDesc& d = bt.d[lo];
    const uint32_t ubase = (chunk - bt.chunk_begin[lo]) * kEwChunk + threadIdx.x;
    if (d.vec > 1) ew_vec<T, kChain>(d, ubase, nf);
    else ew_scalar<T>(d, ubase, nf);
  }
  if (nf) atomicOr(status, kStatusNonFinite);
}

// ------------------------------------------- TMA-staged plain forward ---
// Plain multi-output FQ forward (aligned descriptors): chunks of 1024
// 16-byte units are brought into a kFwdStages-deep shared-memory ring by the
// TMA engine (cp.async.bulk + mbarrier), issued by thread 0 kFwdStages-1
// chunks ahead, so the bytes in flight no longer depend on registers or
// occupancy; threads read conflict-free 16-byte vectors from smem and write
// outputs with 16-byte stores.
constexpr int kFwdChunkBytes = kEwChunk * 16;  // 16 KB

struct ChunkRef {
  int di;
  uint32_t u0;     // first unit of the chunk within the descriptor
  uint32_t units;  // units in this chunk
};

__device__ __forceinline__ ChunkRef locate_chunk(const EwBatch& bt, uint32_t chunk) {
  int lo = 0, hi = bt.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bt.chunk_begin[mid] <= chunk) lo = mid;
    else hi = mid - 1;
  }
  ChunkRef r;
  r.di = lo;
  const uint32_t cu = bt.chunk_units;
  r.u0 = (chunk - bt.chunk_begin[lo]) * cu;
  const uint32_t left = bt.d[lo].nunits - r.u0;
  r.units = left < cu ? left : cu;
  return r;
}

// lean loops enabled (QFB_FWD_LEAN=<mask>, A/B): 1 plain forward, 2 f32
// chains with ReLU / no activation, 4 chains with GELU, 8 binary16 chains
// with ReLU / no activation. Default: all but 2 — the f32 ReLU window is
// memory-bound at 0.95 of HBM on the general loop and the lean loop's
// screens cost it 3-4 % (r02bc); GELU gains 0.73 -> 0.90 (f32), binary16
// ReLU 0.69 -> 0.81 and GELU 0.42 -> 0.54.
// 16: int8 code emission.
constexpr int kLeanPlain = 1, kLeanChain = 2, kLeanChainGelu = 4, kLeanChainHalf = 8, kLeanInt8 = 16;
constexpr int kLeanAll = kLeanPlain | kLeanChain | kLeanChainGelu | kLeanChainHalf | kLeanInt8;
__constant__ int c_fwd_lean = kLeanPlain | kLeanChainGelu | kLeanChainHalf | kLeanInt8;

// ------------------------------------------------ lean plain forward ---
// The plain multi-output forward's per-unit work for the common case (f32,
// no int8 output, no half-grid output, the 3-stage ring), with everything
// loop-invariant hoisted per chunk and the channel's scales recomputed only
// when a thread's unit crosses into a new row (rows are thousands of units
// long). A unit whose values or scales fall outside the shortcut's proven
// domain (f32: the |x| < s * 2^100 screen; f16: inf/NaN, s < 2^-80, or q*s
// beyond the binary16 range) takes fwd_unit_general, the full guarded code,
// out of line. Same bits as the general loop (same functions, same order).
template <typename T>
struct UnitVals {
  float v[Elem<T>::kPerVec];
};

template <typename T>
__device__ __forceinline__ bool fwd_unit_general_body(const EwDesc& d, uint32_t u, uint32_t ch,
                                                      const UnitVals<T>& uv, bool special, bool streaming,
                                                      int jb, int je) {
  constexpr int V = Elem<T>::kPerVec;
  bool nf = false;
  for (int j = jb; j < je; ++j) {
    const float sc = __ldg(d.s[j] + ch);
    const bool fast = fast_div_ok(sc);
    const float rc = fast ? __frcp_rn(sc) : 1.0f;
    float o[V];
    const bool finite = sizeof(T) == 2 ? (!special && fast && sc >= 0x1p-80f)
                                       : (fast && screen_f32<V>(uv.v, __fmul_rn(sc, 0x1p100f)));
    if (finite) {
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = fq_value_fast_finite(uv.v[i], sc, rc, d.q);
    } else if (fast) {
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = fq_value_fast(uv.v[i], sc, rc, d.q);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) o[i] = fq_value(uv.v[i], sc, d.q);
    }
    const bool plain = sizeof(T) == 2 ? (!special && sc * d.q <= 65504.0f) : true;
    const uint4 packed = plain ? Elem<T>::pack_in_range(o) : Elem<T>::pack(o, uv.v, false, nf);
    st_v4(static_cast<uint4*>(d.y[j]) + u, packed, streaming);
  }
  return nf;
}
// out of line for the f32 lean loop; the binary16 lean loop inlines the
// body (a call there raises the kernel's registers from 56 to 76)
template <typename T>
__device__ __noinline__ bool fwd_unit_general(const EwDesc& d, uint32_t u, uint32_t ch, UnitVals<T> uv,
                                              bool special, bool streaming, int jb, int je) {
  return fwd_unit_general_body<T>(d, u, ch, uv, special, streaming, jb, je);
}

// ------------------------------------------------ lean chain loop ---
// Any inf/NaN among a unit's staged values (exponent all ones; the carry
// trick reaches the sign bit of each lane exactly then).
template <typename T>
__device__ __forceinline__ bool nonfinite_unit(const uint4& r) {
  constexpr uint32_t kE = sizeof(T) == 2 ? 0x7c007c00u : 0x7f800000u;
  constexpr uint32_t kOne = sizeof(T) == 2 ? 0x04000400u : 0x00800000u;
  constexpr uint32_t kTop = sizeof(T) == 2 ? 0x80008000u : 0x80000000u;
  return ((((r.x & kE) + kOne) | ((r.y & kE) + kOne) | ((r.z & kE) + kOne) | ((r.w & kE) + kOne)) & kTop) != 0;
}

// qfb_p_gelu for a non-NaN x without branches: the polynomial for every
// element, then the two saturated ranges selected around it (identical
// bits: the middle range runs the same qfb_p_gelu_core).
__device__ __forceinline__ float gelu_nonnan(float x) {
  const float g = qfb_p_gelu_core(x);
  return x > 5.0f ? x : (x < -5.0f ? -0.0f : g);
}

// gelu_nonnan on two lanes with packed f32x2 FMAs for the polynomial: each
// lane runs qfb_p_gelu_core's operations in the same order (IEEE RN per
// lane), the sign selects and the saturated ranges per lane.
__device__ __forceinline__ void gelu2_nonnan(float& a, float& b) {
  const uint64_t u = f2_fma(f2_pack(a < 0.0f ? -a : a, b < 0.0f ? -b : b), f2_pack(0.4f, 0.4f),
                            f2_pack(-1.0f, -1.0f));
  uint64_t h = f2_pack(QFB_P_GELU_C0, QFB_P_GELU_C0);
#define QFB_GELU2_STEP(c) h = f2_fma(h, u, f2_pack(c, c));
  QFB_P_GELU_HORNER(QFB_GELU2_STEP)
#undef QFB_GELU2_STEP
  float ha, hb;
  f2_unpack(h, ha, hb);
  const uint64_t phi = f2_add(f2_pack(0.5f, 0.5f), f2_pack(a < 0.0f ? -ha : ha, b < 0.0f ? -hb : hb));
  float ga, gb;
  f2_unpack(f2_mul(f2_pack(a, b), phi), ga, gb);
  a = a > 5.0f ? a : (a < -5.0f ? -0.0f : ga);
  b = b > 5.0f ? b : (b < -5.0f ? -0.0f : gb);
}

// One chain unit through the general code (x86 NaN propagation, guarded
// quotient, checked binary16 pack): units of the lean chain loop with
// inf/NaN inputs or values outside the screened domain.
template <typename T>
__device__ __noinline__ bool chain_unit_general(const EwDesc& d, uint32_t u, uint32_t ch, uint4 ra, uint4 rb,
                                                bool streaming) {
  constexpr int V = Elem<T>::kPerVec;
  bool nf = false;
  float v[V];
  bool special = Elem<T>::unpack_flag(ra, v);
  if (d.b != nullptr) {
    float w[V];
    special |= Elem<T>::unpack_flag(rb, w);
    if (sizeof(T) == 2 && !special) {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __fadd_rn(v[i], w[i]);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = x86_add(v[i], w[i]);  // tensor.hpp:126-134
    }
  }
  if (d.act != 0) {
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = apply_act(v[i], d.act);
  }
  if (d.flags & kEwDemoteIn) {  // binary16 storage only (the lean loop's domain)
    if (!special) {
#pragma unroll
      for (int i = 0; i < V; i += 2) {
        const float2 f = __half22float2(__floats2half2_rn(fminf(fmaxf(v[i], -65504.0f), 65504.0f),
                                                          fminf(fmaxf(v[i + 1], -65504.0f), 65504.0f)));
        v[i] = f.x;
        v[i + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = half_grid(v[i], v[i], nf);  // tensor.hpp:159-170
    }
  }
  for (int j = 0; j < d.n_out; ++j) {
    const float sc = __ldg(d.s[j] + ch);
    float o[V];
    fq_unit<V>(v, sc, d.q, o);
    const bool plain = sizeof(T) == 2 ? (!special && sc * d.q <= 65504.0f) : true;
    const uint4 packed = plain ? Elem<T>::pack_in_range(o) : Elem<T>::pack(o, v, false, nf);
    st_v4(static_cast<uint4*>(d.y[j]) + u, packed, streaming);
  }
  return nf;
}

// The one-output-at-a-time lean loop for an f32 instance: measured on the
// 2-stage ring (short launches: config-1 map 6.50 -> 5.94 us per call);
// the 3-stage ring keeps its two-output loop (0.1342 vs 0.1349 ms step) and
// the 4-stage ring the general loop (8-frame launches 20.3 k vs 18.5 k
// frames/s with this loop), r02bn.
template <int kFwdStages>
__host__ __device__ constexpr bool one_output_f32() { return kFwdStages == 2; }

// L2 hints (QFB_L2_HINTS mask, A/B): 1 = forward input loads evict_last,
// 16 = only those of the launch's last 4096 chunks (default: one f32 frame
// step 0.1348-0.1351 -> 0.1338-0.1346 ms, forward 53.3 -> 52.7 us, r02bp)
__constant__ int c_l2_hints = 16;

// packed f32x2 FQ arithmetic in the binary16 lean loop (QFB_FQ2=0: scalar, A/B)
__constant__ int c_fq2 = 1;

// V screened values through fq_value_fast_finite, two per FMUL2 / FFMA2
// from their negations (a sign flip each; see fq2_fast_finite_neg)
template <int V>
__device__ __forceinline__ void fq_unit_fast_finite(const float* v, float s, float y, float q, float* o) {
  if (c_fq2) {
    const uint64_t S = f2_pack(s, s), NY = f2_pack(-y, -y);
#pragma unroll
    for (int i = 0; i < V; i += 2) f2_unpack(fq2_fast_finite_neg(f2_pack(-v[i], -v[i + 1]), S, NY, q), o[i], o[i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) o[i] = fq_value_fast_finite(v[i], s, y, q);
  }
}

// The 4-stage ring's general loop takes the screened fast path too, with
// the packed f32x2 quotient: slower in short bursts (8-frame launches
// 20.2 k -> 18.9 k frames/s over 40 launches) but faster in the sustained,
// power-capped run config 5 specifies (32 x 1000 frames: 18.8 k -> 19.8 k),
// where fewer instructions per byte leave more of the power budget to the
// memory system (r02cj, r02ck).
constexpr bool kScreen4 = true;

__device__ __forceinline__ bool lean_enabled(int bit) { return (c_fwd_lean & bit) != 0; }

// kChain: quant -> act -> quant chains (a [+ b] staged, K outputs, optional
// demotion / pre-activation output); 2 arrays per stage, 3 CTAs per SM.
template <typename T, bool kChain, int kFwdStages>
__global__ void __launch_bounds__(kEwThreads, (kChain ? 6 : 10) / kFwdStages)
    ew_tma_kernel(const __grid_constant__ EwBatch bt, uint32_t* __restrict__ status) {
  constexpr int V = Elem<T>::kPerVec;
  constexpr int kArrays = kChain ? 2 : 1;  // a [, b] per stage
  extern __shared__ __align__(128) unsigned char fsmem[];
  uint4* ring = reinterpret_cast<uint4*>(fsmem);
  __shared__ __align__(8) uint64_t bars[kFwdStages];
  __shared__ ChunkRef refs[kFwdStages];
  const int tid = threadIdx.x;

  const uint32_t total = bt.chunk_begin[bt.n];
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x >= total) return;

  // chunks go round robin over the CTAs (consecutive chunks in flight
  // across the grid at any time: a compact, channel-interleaved window)
  auto issue = [&](uint32_t chunk, int s) {
    const ChunkRef r = locate_chunk(bt, chunk);
    const EwDesc& d = bt.d[r.di];
    const bool has_b = kChain && d.b != nullptr;
    refs[s] = r;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&bars[s], r.units * 16u * (has_b ? 2u : 1u));
    uint4* st = ring + s * kArrays * kEwChunk;
    // keep the forward's inputs (bit 1: all; bit 16: the last 4096 chunks =
    // 64 MB, where the backward, visiting its tiles last to first, starts)
    // in L2 for the backward that follows
    if ((c_l2_hints & 1) || ((c_l2_hints & 16) && chunk + 4096u >= total))
      bulk_g2s_hint(st, static_cast<const uint4*>(d.a) + r.u0, r.units * 16u, &bars[s], l2_evict_last());
    else
      bulk_g2s(st, static_cast<const uint4*>(d.a) + r.u0, r.units * 16u, &bars[s]);
    if (has_b) bulk_g2s(st + kEwChunk, static_cast<const uint4*>(d.b) + r.u0, r.units * 16u, &bars[s]);
  };
  if (tid == 0) {
    for (int s = 0; s < kFwdStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
    for (int s = 0; s < kFwdStages - 1; ++s) {
      const uint32_t c = blockIdx.x + (uint32_t)s * gridDim.x;
      if (c < total) issue(c, s);
    }
  }
  __syncthreads();

  bool nf = false;
  uint32_t phase_bits = 0;
  int it = 0;
  for (uint32_t chunk = blockIdx.x; chunk < total; chunk += gridDim.x, ++it) {
    const int s = it % kFwdStages;
    // producer: keep kFwdStages-1 chunks in flight (the target stage was
    // released by the barrier at the end of the previous iteration)
    if (tid == 0) {
      const uint32_t c = chunk + (uint32_t)(kFwdStages - 1) * gridDim.x;
      if (c < total) issue(c, (it + kFwdStages - 1) % kFwdStages);
    }
    mbar_wait(&bars[s], (phase_bits >> s) & 1u);
    phase_bits ^= 1u << s;
    const ChunkRef r = refs[s];
    const EwDesc& d = bt.d[r.di];
    // f16: loop-invariant descriptor fields pinned in registers (the
    // descriptor sits in the dynamically indexed parameter bank and the
    // element-rate-bound f16 loop would re-read it at every use); f32 leaves
    // the choice to the compiler (pinning cost the 4-stage ring 8 %)
    constexpr bool kPin = sizeof(T) == 2;
    FastDivHost pin_inner{};
    uint32_t pin_flags = 0, pin_nout = 0, pin_nch = 0;
    if constexpr (kPin) {
      pin_flags = pin_u(d.flags);
      pin_nout = pin_u((uint32_t)d.n_out);
      pin_inner.d = pin_u(d.inner_u.d);
      pin_inner.m = pin_u(d.inner_u.m);
      pin_inner.s = pin_u(d.inner_u.s);
      pin_nch = pin_u(d.chans.d);
    }
#define QFB_FLAGS (kPin ? pin_flags : d.flags)
#define QFB_NOUT (kPin ? (int)pin_nout : d.n_out)
#define QFB_NCH (kPin ? pin_nch : d.chans.d)
#define QFB_INNER (kPin ? pin_inner : d.inner_u)
    const bool streaming = (QFB_FLAGS & kEwStreaming) != 0;
    const bool half_out = (QFB_FLAGS & kEwHalfGrid) != 0;
    const float qv = pin_f(d.q);
    const uint4* src = ring + s * kArrays * kEwChunk;
    // (f32, 3-stage ring only: the one-frame launches; its registers cost the
    // f16 and the 2/4-stage instances occupancy — measured, r02_as)
    if constexpr (kChain) {
      if (lean_enabled(d.act == 2 ? kLeanChainGelu : sizeof(T) == 2 ? kLeanChainHalf : kLeanChain) &&
          (QFB_FLAGS & (kEwInt8Out | kEwHalfGrid | (sizeof(T) == 2 ? 0u : kEwDemoteIn))) == 0 &&
          d.preact == nullptr) {
        // ---- lean chain loop (no pre-activation output; demotion on
        // binary16 storage only): descriptor fields hoisted, scales
        // reloaded on row crossings, a unit of finite inputs takes the plain
        // add, a branch-free activation, the packed clamped demotion and the
        // screened quotient; anything else goes through chain_unit_general
        // (same functions as the general loop).
        const bool demote = (QFB_FLAGS & kEwDemoteIn) != 0;
        const int nout = (int)pin_u((uint32_t)d.n_out);
        const int act = (int)pin_u((uint32_t)d.act);
        const bool has_b = d.b != nullptr;
        const uint32_t nch = pin_u(d.chans.d);
        FastDivHost inner;
        inner.d = pin_u(d.inner_u.d);
        inner.m = pin_u(d.inner_u.m);
        inner.s = pin_u(d.inner_u.s);
        FastDivHost chans;
        chans.d = nch;
        chans.m = pin_u(d.chans.m);
        chans.s = pin_u(d.chans.s);
        uint4* const y0 = static_cast<uint4*>(d.y[0]);
        uint4* const y1 = static_cast<uint4*>(d.y[1]);
        const float* const s0p = d.s[0];
        const float* const s1p = d.s[1];
        uint32_t row_end = 0, ch = 0;
        float s0 = 1.0f, s1 = 1.0f, r0 = 1.0f, r1 = 1.0f, t0 = 0.0f, t1 = 0.0f;
        bool ok0 = false, ok1 = false;
        for (uint32_t k = tid; k < r.units; k += kEwThreads) {
          const uint32_t u = r.u0 + k;
          if (u >= row_end) {
            const uint32_t row = nch == 1 ? 0u : fdiv(u, inner);
            ch = nch == 1 ? 0u : row - fdiv(row, chans) * nch;
            row_end = nch == 1 ? 0xffffffffu : (row + 1u) * inner.d;
            s0 = __ldg(s0p + ch);
            const bool f0 = fast_div_ok(s0);
            r0 = f0 ? __frcp_rn(s0) : 1.0f;
            t0 = f0 ? __fmul_rn(s0, 0x1p100f) : 0.0f;
            ok0 = f0 && (sizeof(T) == 4 || (s0 >= 0x1p-80f && s0 * qv <= 65504.0f));
            if (nout > 1) {
              s1 = __ldg(s1p + ch);
              const bool f1 = fast_div_ok(s1);
              r1 = f1 ? __frcp_rn(s1) : 1.0f;
              t1 = f1 ? __fmul_rn(s1, 0x1p100f) : 0.0f;
              ok1 = f1 && (sizeof(T) == 4 || (s1 >= 0x1p-80f && s1 * qv <= 65504.0f));
            } else {
              ok1 = true;
              t1 = 0x1p127f;
            }
          }
          const uint4 ra = src[k];
          const uint4 rb = has_b ? src[kEwChunk + k] : make_uint4(0u, 0u, 0u, 0u);
          bool done = false;
          if (!nonfinite_unit<T>(ra) && !(has_b && nonfinite_unit<T>(rb))) {
            float v[V];
            Elem<T>::unpack(ra, v);
            if (has_b) {
              float w[V];
              Elem<T>::unpack(rb, w);
#pragma unroll
              for (int i = 0; i < V; ++i) v[i] = __fadd_rn(v[i], w[i]);  // finite operands: no NaN to propagate
            }
            if (act == 1) {
#pragma unroll
              for (int i = 0; i < V; ++i) v[i] = v[i] > 0.0f ? v[i] : 0.0f;
            } else if (act == 2) {
              if (c_fq2) {
#pragma unroll
                for (int i = 0; i < V; i += 2) gelu2_nonnan(v[i], v[i + 1]);
              } else {
#pragma unroll
                for (int i = 0; i < V; ++i) v[i] = gelu_nonnan(v[i]);
              }
            }
            if (sizeof(T) == 2 && demote) {
              // finite values: round_to_half is the clamped RNE conversion
              // (half.hpp:17-39), two elements per conversion (general loop)
#pragma unroll
              for (int i = 0; i < V; i += 2) {
                const float2 f = __half22float2(__floats2half2_rn(fminf(fmaxf(v[i], -65504.0f), 65504.0f),
                                                                  fminf(fmaxf(v[i + 1], -65504.0f), 65504.0f)));
                v[i] = f.x;
                v[i + 1] = f.y;
              }
            }
            // binary16: the sum of finite halves and its activation stay
            // finite (|a + b| <= 131008), as in the general loop's screen
            const bool fin = sizeof(T) == 2 ? (ok0 && ok1)
                                            : (ok0 && ok1 && screen_f32<V>(v, t0) && screen_f32<V>(v, t1));
            if (fin) {
              float o[V];
              fq_unit_fast_finite<V>(v, s0, r0, qv, o);
              st_v4(y0 + u, Elem<T>::pack_in_range(o), streaming);
              if (nout > 1) {
                fq_unit_fast_finite<V>(v, s1, r1, qv, o);
                st_v4(y1 + u, Elem<T>::pack_in_range(o), streaming);
              }
              done = true;
            }
          }
          if (!done) nf |= chain_unit_general<T>(d, u, ch, ra, rb, streaming);
        }
        __syncthreads();  // stage s free for the producer
        continue;
      }
    }
    if constexpr (!kChain) {
      if (lean_enabled(kLeanInt8) && (QFB_FLAGS & (kEwInt8Out | kEwHalfGrid)) == kEwInt8Out) {
        // ---- lean int8 code emission, one output at a time: a unit whose
        // values pass the screen (f32: |x| < s * 2^100; f16: no inf/NaN and
        // s >= 2^-80) takes the magic-number codes, others code_unit's
        // guarded per-element path (NaN -> 0) — the general loop's functions.
        FastDivHost inner;
        inner.d = pin_u(d.inner_u.d);
        inner.m = pin_u(d.inner_u.m);
        inner.s = pin_u(d.inner_u.s);
        const uint32_t nch = pin_u(d.chans.d);
        FastDivHost chans;
        chans.d = nch;
        chans.m = pin_u(d.chans.m);
        chans.s = pin_u(d.chans.s);
        const int nout = (int)pin_u((uint32_t)d.n_out);
        for (int j = 0; j < nout; ++j) {
          void* const y = d.y[j];
          const float* const sp = d.s[j];
          uint32_t row_end = 0, ch = 0;
          float sj = 1.0f, rj = 1.0f, tj = 0.0f;
          bool fj = false, okj = false;
#pragma unroll 1
          for (uint32_t k = tid; k < r.units; k += kEwThreads) {
            const uint32_t u = r.u0 + k;
            if (u >= row_end) {
              const uint32_t row = nch == 1 ? 0u : fdiv(u, inner);
              ch = nch == 1 ? 0u : row - fdiv(row, chans) * nch;
              row_end = nch == 1 ? 0xffffffffu : (row + 1u) * inner.d;
              sj = __ldg(sp + ch);
              fj = fast_div_ok(sj);
              rj = fj ? __frcp_rn(sj) : 1.0f;
              tj = fj ? __fmul_rn(sj, 0x1p100f) : 0.0f;
              okj = fj && (sizeof(T) == 4 || sj >= 0x1p-80f);
            }
            float v[V];
            const bool special = Elem<T>::unpack_flag(src[k], v);
            const bool fin = sizeof(T) == 2 ? (okj && !special) : screen_f32<V>(v, tj);
            uint32_t c[V];
            if (fin && c_fq2) {
              const uint64_t S = f2_pack(sj, sj), NY = f2_pack(-rj, -rj);
#pragma unroll
              for (int i = 0; i < V; i += 2) code2_fast_finite_neg(f2_pack(-v[i], -v[i + 1]), S, NY, qv, c[i], c[i + 1]);
            } else {
              code_unit<V>(v, sj, rj, fj, qv, c, fin);
            }
            store_codes<V>(y, u, c);
          }
        }
        __syncthreads();  // stage s free for the producer
        continue;
      }
    }
    if constexpr (!kChain && (sizeof(T) == 2 || one_output_f32<kFwdStages>())) {
      if (lean_enabled(kLeanPlain) && (QFB_FLAGS & (kEwInt8Out | kEwHalfGrid)) == 0) {
        // ---- lean loop, one output at a time (binary16, and f32 on the
        // 2-stage ring; the outputs of a two-consumer point re-read the
        // staged unit: a single output's state keeps the loop inside the
        // general loop's registers). A unit outside the shortcut's domain
        // (f32: the |x| < s * 2^100 screen; f16: inf/NaN, s < 2^-80, q*s
        // beyond the binary16 range) takes the general code for that output.
        const uint32_t lnch = pin_u(d.chans.d);
        FastDivHost inner;
        inner.d = pin_u(d.inner_u.d);
        inner.m = pin_u(d.inner_u.m);
        inner.s = pin_u(d.inner_u.s);
        FastDivHost chans;
        chans.d = lnch;
        chans.m = pin_u(d.chans.m);
        chans.s = pin_u(d.chans.s);
        const int lnout = (int)pin_u((uint32_t)d.n_out);
        for (int j = 0; j < lnout; ++j) {
          uint4* const y = static_cast<uint4*>(d.y[j]);
          const float* const sp = d.s[j];
          uint32_t row_end = 0, ch = 0;
          float sj = 1.0f, rj = 1.0f, tj = 0.0f;
          bool ok = false;
#pragma unroll 1
          for (uint32_t k = tid; k < r.units; k += kEwThreads) {
            const uint32_t u = r.u0 + k;
            if (u >= row_end) {  // first unit of the chunk or a new row
              const uint32_t row = lnch == 1 ? 0u : fdiv(u, inner);
              ch = lnch == 1 ? 0u : row - fdiv(row, chans) * lnch;
              row_end = lnch == 1 ? 0xffffffffu : (row + 1u) * inner.d;
              sj = __ldg(sp + ch);
              ok = fast_div_ok(sj) && (sizeof(T) == 4 || (sj >= 0x1p-80f && sj * qv <= 65504.0f));
              rj = ok ? __frcp_rn(sj) : 1.0f;
              tj = ok ? __fmul_rn(sj, 0x1p100f) : 0.0f;
            }
            UnitVals<T> uv;
            const uint4 raw = src[k];
            const bool special = Elem<T>::unpack_flag(raw, uv.v);
            if (sizeof(T) == 2 && c_fq2 && ok && !special) {
              // packed f32x2 quotient from the negated halves (sign flip of
              // the staged words), two elements per FMUL2 / FFMA2
              const uint64_t S = f2_pack(sj, sj), NY = f2_pack(-rj, -rj);
              const uint32_t w[4] = {raw.x ^ 0x80008000u, raw.y ^ 0x80008000u, raw.z ^ 0x80008000u,
                                     raw.w ^ 0x80008000u};
              uint32_t ow[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 nx = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
                float o0, o1;
                f2_unpack(fq2_fast_finite_neg(f2_pack(nx.x, nx.y), S, NY, qv), o0, o1);
                const __half2 h = __floats2half2_rn(o0, o1);
                ow[i] = *reinterpret_cast<const uint32_t*>(&h);
              }
              st_v4(y + u, make_uint4(ow[0], ow[1], ow[2], ow[3]), streaming);
            } else if (sizeof(T) == 2 ? (ok && !special) : screen_f32<V>(uv.v, tj)) {
              float o[V];
              fq_unit_fast_finite<V>(uv.v, sj, rj, qv, o);
              st_v4(y + u, Elem<T>::pack_in_range(o), streaming);
            } else {
              nf |= fwd_unit_general_body<T>(d, u, ch, uv, special, streaming, j, j + 1);
            }
          }
        }
        __syncthreads();  // stage s free for the producer
        continue;
      }
    }
    if constexpr (!kChain && kFwdStages == 3 && sizeof(T) == 4) {
      if (lean_enabled(kLeanPlain) && (QFB_FLAGS & (kEwInt8Out | kEwHalfGrid)) == 0) {
        // ---- lean loop: loop-invariant descriptor fields in registers
        const int nout = (int)pin_u((uint32_t)d.n_out);
        const uint32_t nch = pin_u(d.chans.d);
        FastDivHost inner;
        inner.d = pin_u(d.inner_u.d);
        inner.m = pin_u(d.inner_u.m);
        inner.s = pin_u(d.inner_u.s);
        FastDivHost chans;
        chans.d = nch;
        chans.m = pin_u(d.chans.m);
        chans.s = pin_u(d.chans.s);
        uint4* const y0 = static_cast<uint4*>(d.y[0]);
        uint4* const y1 = static_cast<uint4*>(d.y[1]);
        const float* const s0p = d.s[0];
        const float* const s1p = d.s[1];
        uint32_t row_end = 0, ch = 0;
        float s0 = 1.0f, s1 = 1.0f, r0 = 1.0f, r1 = 1.0f, t0 = 0.0f, t1 = 0.0f;
        bool ok0 = false, ok1 = false;
        for (uint32_t k = tid; k < r.units; k += kEwThreads) {
          const uint32_t u = r.u0 + k;
          if (u >= row_end) {  // first unit of the chunk or a new row
            const uint32_t row = nch == 1 ? 0u : fdiv(u, inner);
            ch = nch == 1 ? 0u : row - fdiv(row, chans) * nch;
            row_end = nch == 1 ? 0xffffffffu : (row + 1u) * inner.d;
            s0 = __ldg(s0p + ch);
            const bool f0 = fast_div_ok(s0);
            r0 = f0 ? __frcp_rn(s0) : 1.0f;
            t0 = f0 ? __fmul_rn(s0, 0x1p100f) : 0.0f;
            ok0 = f0 && (sizeof(T) == 4 || (s0 >= 0x1p-80f && s0 * qv <= 65504.0f));
            if (nout > 1) {
              s1 = __ldg(s1p + ch);
              const bool f1 = fast_div_ok(s1);
              r1 = f1 ? __frcp_rn(s1) : 1.0f;
              t1 = f1 ? __fmul_rn(s1, 0x1p100f) : 0.0f;
              ok1 = f1 && (sizeof(T) == 4 || (s1 >= 0x1p-80f && s1 * qv <= 65504.0f));
            } else {
              ok1 = true;
              t1 = 0x1p127f;
            }
          }
          UnitVals<T> uv;
          const bool special = Elem<T>::unpack_flag(src[k], uv.v);
          const bool fin = sizeof(T) == 2 ? (!special && ok0 && ok1)
                                          : (ok0 && ok1 && screen_f32<V>(uv.v, t0) && screen_f32<V>(uv.v, t1));
          if (fin) {
            float o[V];
            fq_unit_fast_finite<V>(uv.v, s0, r0, qv, o);
            st_v4(y0 + u, Elem<T>::pack_in_range(o), streaming);
            if (nout > 1) {
              fq_unit_fast_finite<V>(uv.v, s1, r1, qv, o);
              st_v4(y1 + u, Elem<T>::pack_in_range(o), streaming);
            }
          } else {
            nf |= fwd_unit_general<T>(d, u, ch, uv, special, streaming, 0, nout);
          }
        }
        __syncthreads();  // stage s free for the producer
        continue;
      }
    }
    // Per-thread scale cache: units of a chunk mostly share a channel, so
    // the channel, its scales and reciprocals are recomputed only when the
    // row changes.
    uint32_t last_row = 0xffffffffu;
    float sc[2] = {1.0f, 1.0f}, rc[2] = {1.0f, 1.0f};
    float thr[2] = {0.0f, 0.0f};  // f32 screen: |x| < s * 2^100 keeps |x * y| < 2^100
    bool fast[2] = {true, true};
    for (uint32_t k = tid; k < r.units; k += kEwThreads) {
      const uint32_t u = r.u0 + k;
      const uint32_t row = QFB_NCH == 1 ? 0u : fdiv(u, QFB_INNER);
      if (row != last_row) {
        last_row = row;
        const uint32_t ch = QFB_NCH == 1 ? 0u : row - fdiv(row, d.chans) * QFB_NCH;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j < QFB_NOUT) {
            sc[j] = __ldg(d.s[j] + ch);
            fast[j] = fast_div_ok(sc[j]);
            rc[j] = fast[j] ? __frcp_rn(sc[j]) : 1.0f;
            thr[j] = fast[j] ? __fmul_rn(sc[j], 0x1p100f) : 0.0f;
          }
        }
      }
      float v[V];
      bool special = Elem<T>::unpack_flag(src[k], v);
      if constexpr (kChain) {
        if (d.b != nullptr) {
          float w[V];
          special |= Elem<T>::unpack_flag(src[kEwChunk + k], w);
          if (sizeof(T) == 2 && !special) {
            // finite binary16 operands: the plain sum (no NaN to propagate)
#pragma unroll
            for (int i = 0; i < V; ++i) v[i] = __fadd_rn(v[i], w[i]);
          } else {
#pragma unroll
            for (int i = 0; i < V; ++i) v[i] = x86_add(v[i], w[i]);  // tensor.hpp:126-134
          }
        }
        if (d.act != 0) {
#pragma unroll
          for (int i = 0; i < V; ++i) v[i] = apply_act(v[i], d.act);
        }
        if (QFB_FLAGS & kEwDemoteIn) {
          if (sizeof(T) == 2 && !special) {
            // finite values (|a + b| <= 131008; ReLU and the portable GELU
            // keep them finite): round_to_half is the clamped RNE conversion
            // (half.hpp:17-39), two elements per conversion
#pragma unroll
            for (int i = 0; i < V; i += 2) {
              const float2 f = __half22float2(__floats2half2_rn(fminf(fmaxf(v[i], -65504.0f), 65504.0f),
                                                                fminf(fmaxf(v[i + 1], -65504.0f), 65504.0f)));
              v[i] = f.x;
              v[i + 1] = f.y;
            }
          } else {
#pragma unroll
            for (int i = 0; i < V; ++i) v[i] = half_grid(v[i], v[i], nf);  // tensor.hpp:159-170
          }
        }
        if (d.preact != nullptr) {
          st_v4(static_cast<uint4*>(d.preact) + u, Elem<T>::pack(v, v, false, nf), streaming);
        }
        // f16 units: finite a, b stay finite through add (|a + b| <= 131008
        // in float), ReLU and the portable GELU, so `special` (inf/NaN in a
        // or b) still selects the guarded FQ and the checked pack; f32 units
        // are always treated as special (no screening)
      }
      if (!kChain && (QFB_FLAGS & kEwInt8Out)) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j >= QFB_NOUT) break;
          uint32_t c[V];
          code_unit<V>(v, sc[j], rc[j], fast[j], qv, c,
                       sizeof(T) == 2 ? (!special && fast[j] && sc[j] >= 0x1p-80f)
                                      : (kFwdStages < 4 && screen_f32<V>(v, thr[j])));
          store_codes<V>(d.y[j], u, c);
        }
        continue;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j >= QFB_NOUT) break;
        float o[V];
        const bool finite = sizeof(T) == 2 ? (!special && fast[j] && sc[j] >= 0x1p-80f)
                                           : ((kFwdStages < 4 || kScreen4) && screen_f32<V>(v, thr[j]));
        if (finite) {
          // binary16 unit without inf/NaN (|x / s| < 2^96) or an f32 unit
          // passing the screen: no guards needed
          if constexpr (kScreen4 && kFwdStages == 4) {
            fq_unit_fast_finite<V>(v, sc[j], rc[j], qv, o);
          } else {
#pragma unroll
            for (int i = 0; i < V; ++i) o[i] = fq_value_fast_finite(v[i], sc[j], rc[j], qv);
          }
        } else if (fast[j]) {
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = fq_value_fast(v[i], sc[j], rc[j], qv);
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) o[i] = fq_value(v[i], sc[j], qv);
        }
        // f16 store: FQ outputs of finite inputs are bounded by q*s; when
        // that is within the half range a plain packed conversion is exact
        const bool plain = sizeof(T) == 2 ? (!special && sc[j] * qv <= 65504.0f) : !half_out;
        const uint4 packed = plain ? Elem<T>::pack_in_range(o) : Elem<T>::pack(o, v, half_out, nf);
        st_v4(static_cast<uint4*>(d.y[j]) + u, packed, streaming);
      }
    }
#undef QFB_FLAGS
#undef QFB_NOUT
#undef QFB_NCH
#undef QFB_INNER
    __syncthreads();  // stage s free for the producer
  }
  if (nf) atomicOr(status, kStatusNonFinite);
}

// ------------------------------------------------------------ codes ---
template <typename T>
__global__ void __launch_bounds__(kEwThreads) codes_kernel(const __grid_constant__ CodesDesc d) {
  constexpr int V = Elem<T>::kPerVec;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < d.nunits; u += stride) {
    const uint32_t ch = channel_of(u, d.inner_u, d.chans);
    const float s = __ldg(d.s + ch);
    if (d.vec > 1) {
      float v[V];
      Elem<T>::unpack(ld_nc_v4(static_cast<const uint4*>(d.x) + u), v);
      uint32_t w[V / 4];
#pragma unroll
      for (int i = 0; i < V / 4; ++i) {
        w[i] = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          w[i] |= (uint32_t)(uint8_t)fq_code(v[4 * i + b], s, d.q) << (8 * b);
      }
      if (V == 4) {
        reinterpret_cast<uint32_t*>(d.codes)[u] = w[0];
      } else {
        reinterpret_cast<uint2*>(d.codes)[u] = make_uint2(w[0], w[V / 4 - 1]);
      }
    } else {
      d.codes[u] = fq_code(Elem<T>::load1(d.x, u), s, d.q);
    }
  }
}

// --------------------------------------------------- per-operator ---
// exec.hpp:276-342: four sweeps, float temporaries. op0 reads dtype,
// op3 writes dtype (with the half re-round of exec.hpp:306-307).
template <typename T, int OP>
__global__ void __launch_bounds__(kEwThreads)
    perop_kernel(const __grid_constant__ PerOpDesc d, uint32_t* __restrict__ status) {
  bool nf = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d.n; i += stride) {
    const uint64_t ch = d.chans == 1 ? 0 : (i / d.inner) % d.chans;
    // NaNs are carried through the temporaries with the input's sign, as
    // the host reference does, so a half re-round in op 3 sees the same sign.
    if (OP == 0) {
      const float x = Elem<T>::load1(d.in, i);
      static_cast<float*>(d.out)[i] =
          isnan(x) ? __uint_as_float(__float_as_uint(x) | 0x400000u) : __fdiv_rn(x, __ldg(d.s + ch));
    } else if (OP == 1) {
      static_cast<float*>(d.out)[i] = fq_clip(static_cast<const float*>(d.in)[i], d.q);
    } else if (OP == 2) {
      const float c = static_cast<const float*>(d.in)[i];
      static_cast<float*>(d.out)[i] = isnan(c) ? c : rintf(c);
    } else {
      const float r = static_cast<const float*>(d.in)[i];
      const float v = isnan(r) ? r : __fmul_rn(__ldg(d.s + ch), r);
      // sign source: NaN results come from a NaN input; r carries its sign
      Elem<T>::store1(d.out, i, v, r, (d.flags & kEwHalfGrid) != 0, nf);
    }
  }
  if (nf) atomicOr(status, kStatusNonFinite);
}

// ------------------------------------------------------------- rng ---
// rng.hpp:15-50, identical integer/double arithmetic.
__device__ __forceinline__ uint64_t smix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <typename T>
__global__ void fill_rng_kernel(T* out, int64_t n, uint64_t seed_mix, uint64_t stream_term,
                                uint64_t offset, int kind, double lo, double hi) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t idx = offset + (uint64_t)i;
    double v;
    if (kind == 0) {
      const uint64_t w = smix(seed_mix ^ smix(stream_term + idx));
      const double u = __dmul_rn((double)(w >> 11), 0x1.0p-53);
      v = __dadd_rn(lo, __dmul_rn(__dadd_rn(hi, -lo), u));
    } else {
      double acc = 0.0;
      for (uint64_t k = 0; k < 12; ++k) {
        const uint64_t w = smix(seed_mix ^ smix(stream_term + idx * 12 + k));
        acc = __dadd_rn(acc, __dmul_rn((double)(w >> 11), 0x1.0p-53));
      }
      v = __dmul_rn(lo, __dadd_rn(acc, -6.0));
    }
    const float f = __double2float_rn(v);
    if constexpr (sizeof(T) == 4) {
      out[i] = f;
    } else {
      bool nf = false;
      out[i] = half_store(f, f, nf);
    }
  }
}

// ------------------------------------------------------- resolve ---
// quant.hpp:71-109 and :241-244 with the CUDA double libm (the paper's
// scale kernel). May differ from glibc by <= 1-2 ulp.
__global__ void resolve_kernel(const __grid_constant__ ResolveDesc d, uint32_t* status) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  const double ls = d.log_s[i];
  if (!isfinite(ls)) {
    atomicOr(status, kStatusNonFinite);
    return;
  }
  const double sp = ls > 30.0 ? ls + log1p(exp(-ls)) : log1p(exp(ls));
  const double raw = sp + d.eps;
  double s = raw < d.lo ? d.lo : raw;
  s = d.s_max < s ? d.s_max : s;
  if (d.s32) d.s32[i] = (float)s;
  if (d.s64) d.s64[i] = s;
  if (d.chain) {
    const bool clamped = !(raw > d.lo && raw < d.s_max);
    double sg;
    if (ls >= 0.0) {
      sg = 1.0 / (1.0 + exp(-ls));
    } else {
      const double e = exp(ls);
      sg = e / (1.0 + e);
    }
    d.chain[i] = clamped ? 0.0 : sg;
  }
}

}  // namespace

size_t ew_tma_smem(bool chain, int stages) { return (size_t)stages * kFwdChunkBytes * (chain ? 2 : 1); }

template <typename T, bool kChain>
static const void* tma_fn_c(int stages) {
  switch (stages) {
    case 3: return (const void*)ew_tma_kernel<T, kChain, 3>;
    case 4: return (const void*)ew_tma_kernel<T, kChain, 4>;
    default: return (const void*)ew_tma_kernel<T, kChain, 2>;
  }
}

static const void* tma_fn(int dtype, bool chain, int stages) {
  if (dtype == 0) return chain ? tma_fn_c<float, true>(stages) : tma_fn_c<float, false>(stages);
  return chain ? tma_fn_c<__half, true>(stages) : tma_fn_c<__half, false>(stages);
}

cudaError_t ew_tma_occupancy(int dtype, bool chain, int stages, int* blocks_per_sm) {
  const void* f = tma_fn(dtype, chain, stages);
  const int smem = (int)ew_tma_smem(chain, stages);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, kEwThreads, smem);
}

cudaError_t launch_ew_tma(int dtype, bool chain, int stages, const EwBatch& b, uint32_t* status,
                          int grid, cudaStream_t st, bool small) {
  static const cudaError_t lean_set = [] {
    const char* e = getenv("QFB_FWD_LEAN");
    if (!(e && e[0])) return cudaSuccess;
    const int mask = (int)strtol(e, nullptr, 0) & kLeanAll;
    return cudaMemcpyToSymbol(c_fwd_lean, &mask, sizeof mask);
  }();
  if (lean_set != cudaSuccess) return lean_set;
  static const cudaError_t hints_set = [] {
    const char* e = getenv("QFB_L2_HINTS");
    if (!(e && e[0])) return cudaSuccess;
    const int mask = (int)strtol(e, nullptr, 0);
    return cudaMemcpyToSymbol(c_l2_hints, &mask, sizeof mask);
  }();
  if (hints_set != cudaSuccess) return hints_set;
  static const cudaError_t fq2_set = [] {
    const char* e = getenv("QFB_FQ2");
    if (!(e && e[0] == '0')) return cudaSuccess;
    const int off = 0;
    return cudaMemcpyToSymbol(c_fq2, &off, sizeof off);
  }();
  if (fq2_set != cudaSuccess) return fq2_set;
  void* args[] = {const_cast<EwBatch*>(&b), &status};
  return launch_main(tma_fn(dtype, chain, stages), dim3(grid), dim3(kEwThreads), args,
                     ew_tma_smem(chain, stages), st, small ? (kPdlFwd | kPdlFwdSmall) : kPdlFwd);
}

cudaError_t launch_ew(int dtype, bool chain, const EwBatch& b, uint32_t* status, int grid,
                      cudaStream_t st) {
  if (chain) {
    if (dtype == 0) ew_kernel<float, true><<<grid, kEwThreads, 0, st>>>(b, status);
    else ew_kernel<__half, true><<<grid, kEwThreads, 0, st>>>(b, status);
  } else {
    if (dtype == 0) ew_kernel<float, false><<<grid, kEwThreads, 0, st>>>(b, status);
    else ew_kernel<__half, false><<<grid, kEwThreads, 0, st>>>(b, status);
  }
  return cudaGetLastError();
}

cudaError_t launch_codes(int dtype, const CodesDesc& d, int grid, cudaStream_t st) {
  if (dtype == 0) codes_kernel<float><<<grid, kEwThreads, 0, st>>>(d);
  else codes_kernel<__half><<<grid, kEwThreads, 0, st>>>(d);
  return cudaGetLastError();
}

template <typename T>
static void perop_dispatch(int op, const PerOpDesc& d, uint32_t* status, int grid,
                           cudaStream_t st) {
  switch (op) {
    case 0: perop_kernel<T, 0><<<grid, kEwThreads, 0, st>>>(d, status); break;
    case 1: perop_kernel<T, 1><<<grid, kEwThreads, 0, st>>>(d, status); break;
    case 2: perop_kernel<T, 2><<<grid, kEwThreads, 0, st>>>(d, status); break;
    default: perop_kernel<T, 3><<<grid, kEwThreads, 0, st>>>(d, status); break;
  }
}

cudaError_t launch_perop(int dtype, int op, const PerOpDesc& d, uint32_t* status, int grid,
                         cudaStream_t st) {
  if (dtype == 0) perop_dispatch<float>(op, d, status, grid, st);
  else perop_dispatch<__half>(op, d, status, grid, st);
  return cudaGetLastError();
}

cudaError_t launch_fill_rng(int dtype, void* out, int64_t n, uint64_t seed, uint64_t stream,
                            uint64_t offset, int kind, double lo, double hi, int grid,
                            cudaStream_t st) {
  // word(i) = mix(mix(seed ^ K) ^ mix(stream * G + i)), rng.hpp:29-32
  const uint64_t seed_mix = [] (uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
  }(seed ^ 0x243f6a8885a308d3ull);
  const uint64_t stream_term = stream * 0x9e3779b97f4a7c15ull;
  if (dtype == 0)
    fill_rng_kernel<float><<<grid, 256, 0, st>>>(static_cast<float*>(out), n, seed_mix,
                                                 stream_term, offset, kind, lo, hi);
  else
    fill_rng_kernel<__half><<<grid, 256, 0, st>>>(static_cast<__half*>(out), n, seed_mix,
                                                  stream_term, offset, kind, lo, hi);
  return cudaGetLastError();
}

cudaError_t launch_resolve(const ResolveDesc& d, uint32_t* status, cudaStream_t st) {
  const int threads = 128;
  const int grid = (int)((d.n + threads - 1) / threads);
  if (grid > 0) resolve_kernel<<<grid, threads, 0, st>>>(d, status);
  return cudaGetLastError();
}

}  // namespace qfb

namespace qfb {
// Occupancy of the elementwise kernel (sizes the persistent grid).
cudaError_t ew_occupancy(int dtype, bool chain, int* blocks_per_sm) {
  const void* f = chain ? (dtype == 0 ? (const void*)ew_kernel<float, true> : (const void*)ew_kernel<__half, true>)
                        : (dtype == 0 ? (const void*)ew_kernel<float, false> : (const void*)ew_kernel<__half, false>);
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, f, kEwThreads, 0);
}
}  // namespace qfb
