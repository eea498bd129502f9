// qfb_device.cuh — device-side scalar contract of the fake-quant path.
//
// Every function here restates one reference scalar operation bit-exactly
// (paths relative to /root/reference/proj/include/quantfuse/). Compiled
// without fast-math, with FTZ off and IEEE division (nvcc defaults); the
// arithmetic that must not be contracted is spelled with _rn intrinsics.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "qfb_kernels.h"

namespace qfb {

// Status latch bits (qfb_ctx_sync maps them to qfb_status).
constexpr uint32_t kStatusNonFinite = 1u;

// ---------------------------------------------------------------- FQ ---
// quant.hpp:114-121:  s * nearbyintf(min(max(x / s, -q), q))
//  - IEEE round-to-nearest division (__fdiv_rn), never x * (1/s);
//  - the clip is a pair of compare-selects exactly like std::max/std::min,
//    so NaN propagates (fmaxf/fminf would drop it);
//  - rintf == nearbyintf under round-to-nearest-even (FRND);
//  - the product keeps the sign of zero (no integer round trip).
__device__ __forceinline__ float fq_clip(float z, float q) {
  z = (z < -q) ? -q : z;  // std::max(z, -q)
  z = (q < z) ? q : z;    // std::min(z, q)
  return z;
}

// x86 NaN propagation (the reference's host semantics): an operation with
// one NaN operand returns that operand quieted (sign and payload kept); an
// invalid operation (inf - inf, 0 * inf) returns the x86 default NaN
// 0xffc00000. The GPU instead returns a canonical 0x7fffffff, so the paths
// whose NaN bits are observable emulate the host rule explicitly.
__device__ __forceinline__ float quiet_nan(float v) {
  return __uint_as_float(__float_as_uint(v) | 0x400000u);
}
constexpr uint32_t kX86DefaultNaN = 0xffc00000u;

__device__ __forceinline__ float x86_add(float a, float b) {
  const float r = __fadd_rn(a, b);
  if (!isnan(r)) return r;
  return isnan(a) ? quiet_nan(a) : isnan(b) ? quiet_nan(b) : __uint_as_float(kX86DefaultNaN);
}

// NaN in -> the same NaN (quieted) out, exactly as x/s, the selects,
// nearbyintf and s*r propagate it on the host.
__device__ __forceinline__ float fq_value(float x, float s, float q) {
  if (isnan(x)) return quiet_nan(x);
  const float z = __fdiv_rn(x, s);
  return __fmul_rn(s, rintf(fq_clip(z, q)));
}

// Division shortcut for the hot forward: Markstein-corrected quotient with
// a hoisted correctly rounded reciprocal y = __frcp_rn(s) — one FMUL + two
// FFMA per element instead of MUFU.RCP + refinement + FCHK + branch.
// Bit-identical to __fdiv_rn for every normal x, s with a normal quotient:
// proven by exhaustion over all 2^46 significand pairs (tools/verify_div.cu,
// result in profiles/).
__device__ __forceinline__ float markstein_div(float x, float s, float y) {
  const float q0 = __fmul_rn(x, y);
  const float r = __fmaf_rn(-s, q0, x);
  return __fmaf_rn(r, y, q0);
}

// Scales for which the shortcut is used (y finite and normal).
__device__ __forceinline__ bool fast_div_ok(float s) {
  return s >= 0x1p-100f && s <= 0x1p100f;
}

// fq_value via the shortcut; requires fast_div_ok(s) and y = __frcp_rn(s).
// Outside the proven range the quotient only feeds rint(clip(.)):
//  - |q0| >= 2^100 (incl. inf): clip saturates to +-q for both paths;
//  - subnormal/tiny quotients: |z| < 0.5 rounds to +-0 for both paths, and
//    copysign restores the sign of x that FMA-based correction can lose on
//    signed zeros. tools/verify_div.cu test 2 checks every 2^32 x.
// Branch-free: a NaN x runs the arithmetic on garbage (the min/max clip
// drops NaN) and the final select returns the quieted input, exactly what
// the host's NaN propagation yields.
__device__ __forceinline__ float fq_value_fast(float x, float s, float y, float q) {
  const float q0 = __fmul_rn(x, y);
  float z = __fmaf_rn(__fmaf_rn(-s, q0, x), y, q0);
  z = fabsf(q0) < 0x1p100f ? z : q0;
  z = copysignf(z, x);
  z = fminf(fmaxf(z, -q), q);  // == the compare-select clip for non-NaN z
  const float r = __fmul_rn(s, rintf(z));
  return isnan(x) ? quiet_nan(x) : r;
}

// fq_value_fast for a finite, non-NaN x with |x * y| < 2^100 (binary16
// inputs, |x| <= 65504, with s >= 2^-80): the overflow guard and the NaN
// select of fq_value_fast are identities there and are dropped.
// The residual is formed negated, r' = s*q0 - x (= -(x - s*q0) exactly,
// RN being symmetric), and z = q0 - r'*y: the same value as the positive
// form for every x != 0, and for x = +-0 it yields +-0 with x's sign
// (-0: r' = -0 + +0 = +0, z = -0 + -0 = -0), so no copysign is needed.
// tests/test_gpu_fwd.py::test_half_fast_path_all_values checks every
// finite binary16 x over 64 scales; tools/verify_div.cu test 2b every f32
// x with |x| < s * 2^100 (the f32 screen) over 192 scales.
__device__ __forceinline__ float fq_value_fast_finite(float x, float s, float y, float q) {
  const float q0 = __fmul_rn(x, y);
  float z = __fmaf_rn(-__fmaf_rn(s, q0, -x), y, q0);
  z = fminf(fmaxf(z, -q), q);
  return __fmul_rn(s, rintf(z));
}

// Packed f32x2 arithmetic (sm_100 FMUL2 / FFMA2: two IEEE round-to-nearest
// float operations per instruction, denormals kept — no .ftz).
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// fq_value_fast_finite on two values at once, from their NEGATIONS nx = -x
// (free in the binary16 unpack: a sign flip of the packed word): with
// NY = (-y, -y) and S = (s, s), q0 = RN(nx * -y) = RN(x*y), r' = RN(s*q0 +
// nx) = RN(s*q0 - x), z = RN(r' * -y + q0) = RN(q0 - r'*y) — operation for
// operation the scalar function's values (x = +-0 included), then the
// clamp and rint per lane and the product s * rint(z) packed again.
__device__ __forceinline__ uint64_t fq2_fast_finite_neg(uint64_t nx, uint64_t S, uint64_t NY, float q) {
  const uint64_t q0 = f2_mul(nx, NY);
  const uint64_t r = f2_fma(S, q0, nx);
  const uint64_t z = f2_fma(r, NY, q0);
  float z0, z1;
  f2_unpack(z, z0, z1);
  z0 = rintf(fminf(fmaxf(z0, -q), q));
  z1 = rintf(fminf(fmaxf(z1, -q), q));
  return f2_mul(S, f2_pack(z0, z1));
}

// fq_code_bits_fast_finite on two values from their negations (the
// quotient as in fq2_fast_finite_neg, clamp per lane, the magic-number
// round into the low byte as one packed add).
__device__ __forceinline__ void code2_fast_finite_neg(uint64_t nx, uint64_t S, uint64_t NY, float q, uint32_t& c0,
                                                      uint32_t& c1) {
  const uint64_t q0 = f2_mul(nx, NY);
  const uint64_t r = f2_fma(S, q0, nx);
  float z0, z1;
  f2_unpack(f2_fma(r, NY, q0), z0, z1);
  z0 = fminf(fmaxf(z0, -q), q);
  z1 = fminf(fmaxf(z1, -q), q);
  float b0, b1;
  f2_unpack(f2_add(f2_pack(z0, z1), f2_pack(12582912.0f, 12582912.0f)), b0, b1);
  c0 = __float_as_uint(b0);
  c1 = __float_as_uint(b1);
}

// int8 code bits (low byte) of a screened finite x (|x| < s * 2^100, no
// NaN): negated-residual quotient, clip, and round-to-nearest-even into the
// low byte by adding 1.5 * 2^23 (|z| <= q). Equals fq_code
// (tools/verify_div.cu test 2b, all 2^32 x).
__device__ __forceinline__ uint32_t fq_code_bits_fast_finite(float x, float s, float y, float q) {
  const float q0 = __fmul_rn(x, y);
  float z = __fmaf_rn(-__fmaf_rn(s, q0, -x), y, q0);
  z = fminf(fmaxf(z, -q), q);
  return __float_as_uint(__fadd_rn(z, 12582912.0f));
}

// Pin a uniform in a register (stops rematerialization from the
// dynamically indexed parameter bank at every use).
__device__ __forceinline__ float pin_f(float v) {
  float r;
  asm volatile("mov.b32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ uint32_t pin_u(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// ----------------------------------------------------------- binary16 ---
// half.hpp:72-82 round_to_half: |v| > 65504 saturates to +-65504 (never
// inf); NaN maps to +-65504 through the exponent guard of f32_to_f16_rne
// (half.hpp:24-26) with the sign of the NaN. On the device a NaN produced
// by arithmetic is canonical (+), while the host propagates the operand's
// sign, so callers pass the sign source (the offending input).
// For non-NaN v: RNE(clamp(v)) == __float2half_rn(clamp(v)) for every float
// (verified exhaustively).
__device__ __forceinline__ __half half_store(float v, float sign_src, bool& nonfinite) {
  if (!isfinite(v)) nonfinite = true;
  if (isnan(v)) return __ushort_as_half(signbit(sign_src) ? 0xfbffu : 0x7bffu);
  v = fminf(fmaxf(v, -65504.0f), 65504.0f);
  return __float2half_rn(v);
}

__device__ __forceinline__ float half_grid(float v, float sign_src, bool& nonfinite) {
  return __half2float(half_store(v, sign_src, nonfinite));
}

// ---------------------------------------------------- int8 code ---
// quant.hpp:186: static_cast<int8_t>(nearbyintf(clip(x/s))). NaN -> 0
// (the x86 reference truncates through int32 0x80000000, low byte 0).
__device__ __forceinline__ int8_t fq_code(float x, float s, float q) {
  const float r = rintf(fq_clip(__fdiv_rn(x, s), q));
  const int32_t w = isnan(r) ? 0 : __float2int_rz(r);
  return (int8_t)(uint8_t)(uint32_t)w;
}

// ----------------------------------------------- STE / LSQ terms ---
// quant.hpp:217-228 in double: z = x/s, mask = |z| <= q,
// d_ds = mask ? rint(z) - z : (z > 0 ? q : -q).
// d_input = float(mask * double(up)) with host NaN rules: NaN upstream
// propagates (quieted); a masked-out inf gives 0*inf = default NaN.
__device__ __forceinline__ float masked_upstream(bool mask, float up) {
  const uint32_t ub = __float_as_uint(up);
  float d = mask ? up : __uint_as_float(ub & 0x80000000u);  // +-0 with the sign of up
  if ((ub & 0x7f800000u) == 0x7f800000u) {                   // inf / NaN (rare)
    d = (ub & 0x7fffffu) ? quiet_nan(up) : (mask ? up : __uint_as_float(kX86DefaultNaN));
  }
  return d;
}

struct GradTerm {
  bool mask;
  double d_ds;
};

__device__ __forceinline__ GradTerm grad_term(float x, double s, double q) {
  const double z = __ddiv_rn((double)x, s);
  GradTerm t;
  t.mask = fabs(z) <= q;
  t.d_ds = t.mask ? __dadd_rn(rint(z), -z) : (z > 0.0 ? q : -q);
  return t;
}

// Fast double division for the backward: z = RN(x / s) for float x from a
// hoisted y = RN(1/s) per tile (markstein2_div below).
struct DivCtx {
  double s;
  double y;     // RN(1/s)
  double ylo;   // RN(RN(1 - s*y) * y): y + ylo = 1/s to ~2^-105 (markstein_dd only)
  bool usable;  // s in [2^-100, 2^100]
};

__device__ __forceinline__ DivCtx make_div(double s) {
  DivCtx c;
  c.s = s;
  c.y = __drcp_rn(s);
  c.usable = s >= 0x1p-100 && s <= 0x1p100;
  return c;
}

// Two Markstein corrections from the hoisted y = RN(1/s): the first makes
// the quotient faithful (|q0 - x/s| <= 2 ulp, and q0 + r0*y lies within
// 2^-52 ulp of x/s before rounding), and Markstein's theorem (y = RN(1/s),
// z1 within one ulp of x/s => RN(z1 + (x - s*z1)*y) = RN(x/s), no
// underflow/overflow) makes the second correctly rounded. Valid for every
// finite float x (zeros give +-0, whose sign the callers do not observe)
// and s in [2^-100, 2^100] (DivCtx::usable). Validated against __ddiv_rn
// for all 2^32 float x and 40,290 scales (tools/verify_ddiv2.cu,
// profiles/r01_verify_ddiv2.txt: 0 mismatches).
__device__ __forceinline__ double markstein2_div(double x, const DivCtx& c) {
  const double q0 = __dmul_rn(x, c.y);
  const double z1 = __fma_rn(__fma_rn(-c.s, q0, x), c.y, q0);
  return __fma_rn(__fma_rn(-c.s, z1, x), c.y, z1);
}

// Low half of the double-double reciprocal: 1 - s*y is exact (FMA residual
// of the correctly rounded reciprocal), times y ~ (1/s - y).
__device__ __forceinline__ double recip_lo(double s, double y) { return __dmul_rn(__fma_rn(-s, y, 1.0), y); }

// z = RN(x / s) from the double-double reciprocal (y, ylo) and ONE
// Markstein correction: q0 = RN(x*y + RN(x*ylo)) is within 1/2 ulp +
// 2^-103 |x/s| of x/s (faithful), so z = RN(q0 + (x - s*q0)*y) is the
// correctly rounded quotient (y = RN(1/s), q0 faithful: Markstein's
// theorem). Four FP64 ops at dependency depth 4 (markstein2_div: five,
// depth 5). Same domain as markstein2_div (s in [2^-100, 2^100], finite
// x; inf/NaN x give NaN). Validated against __ddiv_rn for all 2^32 float x
// and 40,290 scales (tools/verify_ddiv3.cu, profiles/r02_verify_ddiv3.txt).
__device__ __forceinline__ double markstein_dd(double x, const DivCtx& c) {
  const double q0 = __fma_rn(x, c.y, __dmul_rn(x, c.ylo));
  return __fma_rn(__fma_rn(-c.s, q0, x), c.y, q0);
}

// ------------------------------------------------------ fast divide ---
// Unsigned 32-bit division by a runtime-invariant divisor (round-up
// multiplier method); exact for every n < 2^32.
using FastDiv = FastDivHost;

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  if (f.d == 1) return n;
  const uint32_t hi = __umulhi(n, f.m);
  return (uint32_t)(((uint64_t)hi + n) >> f.s);
}

// -------------------------------------------------------- memory ---
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v, bool streaming) {
  if (streaming) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  } else {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  }
}

// ------------------------------------------- TMA bulk copy + mbarrier ---
// 1-D bulk async copies (cp.async.bulk, the TMA engine without a tensor
// map) into shared memory, completion tracked by an mbarrier transaction
// count. Addresses and sizes must be 16-byte aligned / multiples of 16.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Orders this thread's generic-proxy shared accesses (after a CTA barrier:
// everyone's) before subsequent async-proxy (bulk copy) writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 eviction-priority policies for the cache-hinted bulk copies.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes), "l"(pol)
               : "memory");
}
// Bulk store shared -> global (cp.async.bulk, bulk-group completion).
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// Bulk prefetch of [src, src + bytes) into L2 (no shared memory, no
// completion tracking): src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// Wait until all committed bulk stores have finished READING shared memory.
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// Wait until all committed bulk stores are complete (visible in global).
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// LSU-path async copy (16 bytes, L2 only) and its mbarrier completion hook:
// the arrive fires once all of this thread's prior cp.async have landed.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Programmatic dependent launch (see qfb_kernels.h launch_main): wait for
// the preceding grid (no-op without the launch attribute) / let the next
// one be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// try_wait with a suspend-time hint: the waiting warp is parked by the
// hardware until the phase completes (or the hint expires) instead of
// spinning through issue slots the computing warps need.
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(0x100000u)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_sleep(bar, parity)) {
  }
}

// Element <-> float conversions for the two storage types. A "unit" is
// one 16-byte vector: 4 floats or 8 halves.
template <typename T>
struct Elem;

template <>
struct Elem<float> {
  static constexpr int kPerVec = 4;
  __device__ __forceinline__ static bool unpack_flag(const uint4& r, float* v) {
    unpack(r, v);
    return true;  // not tracked for f32: callers take the general pack
  }
  __device__ __forceinline__ static uint4 pack_in_range(const float* v) {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
  }
  __device__ __forceinline__ static void unpack(const uint4& r, float* v) {
    v[0] = __uint_as_float(r.x);
    v[1] = __uint_as_float(r.y);
    v[2] = __uint_as_float(r.z);
    v[3] = __uint_as_float(r.w);
  }
  // half_grid: re-round onto the binary16 grid (EmulatedHalf in f32).
  __device__ __forceinline__ static uint4 pack(const float* v, const float* sign_src,
                                               bool half_grid_out, bool& nf) {
    float o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = half_grid_out ? half_grid(v[i], sign_src[i], nf) : v[i];
    return make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]),
                      __float_as_uint(o[3]));
  }
  __device__ __forceinline__ static float load1(const void* p, uint64_t i) {
    return __ldg(static_cast<const float*>(p) + i);
  }
  __device__ __forceinline__ static void store1(void* p, uint64_t i, float v, float sign_src,
                                                bool half_grid_out, bool& nf) {
    static_cast<float*>(p)[i] = half_grid_out ? half_grid(v, sign_src, nf) : v;
  }
};

// binary16 bits -> float bits with NaN sign/payload kept (f16_to_f32,
// half.hpp:62-63); the hardware conversion returns a canonical NaN.
__device__ __forceinline__ float half_bits_to_float_exact(uint32_t h) {
  const float f = __half2float(__ushort_as_half((unsigned short)h));
  if ((h & 0x7c00u) == 0x7c00u && (h & 0x3ffu))
    return __uint_as_float(((h & 0x8000u) << 16) | 0x7f800000u | ((h & 0x3ffu) << 13));
  return f;
}

template <>
struct Elem<__half> {
  static constexpr int kPerVec = 8;
  // Returns true when the unit holds an inf/NaN (all-ones exponent).
  __device__ __forceinline__ static bool unpack_flag(const uint4& r, float* v) {
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
    // rare path: any all-ones exponent (inf/NaN) in the unit. Per 16-bit
    // half, (h & 0x7c00) + 0x0400 reaches bit 15 exactly when the exponent
    // is all ones, and never carries into the other half of the word.
    constexpr uint32_t kE = 0x7c007c00u, kOne = 0x04000400u;
    const uint32_t e = (((r.x & kE) + kOne) | ((r.y & kE) + kOne) | ((r.z & kE) + kOne) |
                        ((r.w & kE) + kOne)) & 0x80008000u;
    if (e) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v[2 * i] = half_bits_to_float_exact(w[i] & 0xffffu);
        v[2 * i + 1] = half_bits_to_float_exact(w[i] >> 16);
      }
    }
    return e != 0;
  }
  __device__ __forceinline__ static void unpack(const uint4& r, float* v) { (void)unpack_flag(r, v); }
  // Finite values known to lie within +-65504: plain packed RNE conversion.
  __device__ __forceinline__ static uint4 pack_in_range(const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  // f16 storage always rounds through half_store (RNE + saturation).
  __device__ __forceinline__ static uint4 pack(const float* v, const float* sign_src,
                                               bool /*half_grid_out*/, bool& nf) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t lo = __half_as_ushort(half_store(v[2 * i], sign_src[2 * i], nf));
      const uint32_t hi = __half_as_ushort(half_store(v[2 * i + 1], sign_src[2 * i + 1], nf));
      w[i] = lo | (hi << 16);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  __device__ __forceinline__ static float load1(const void* p, uint64_t i) {
    return half_bits_to_float_exact(static_cast<const unsigned short*>(p)[i]);
  }
  __device__ __forceinline__ static void store1(void* p, uint64_t i, float v, float sign_src,
                                                bool /*half_grid_out*/, bool& nf) {
    static_cast<__half*>(p)[i] = half_store(v, sign_src, nf);
  }
};

}  // namespace qfb
