/*
 * qf_oracle.c — CPU restatement of the reference fake-quant path.
 *
 * TEST INFRASTRUCTURE ONLY (see qf_oracle.h). Written from the reference's
 * stated algorithm; every function cites the reference lines it restates
 * (paths relative to /root/reference/proj/include/quantfuse/).
 *
 * Build: gcc -std=c11 -O2 -ffp-contract=off -fno-fast-math (oracle/Makefile).
 * No -march: like the reference's own Release build, nearbyintf/rintf and
 * fmaf resolve to the correctly rounded libm routines.
 */
#include "qf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../include/qfb_portable.h"

/* ---------------------------------------------------------------- config */

/* quant.hpp:35-43 defaults. */
void orc_cfg_default(orc_cfg* c) {
  c->bits = 8;
  c->reserved = 0;
  c->s_min = 1e-6;
  c->s_min_half = 1e-4;
  c->s_max = 64.0;
  c->eps = 1e-8;
}

/* quant.hpp:49-60. */
int orc_cfg_validate(const orc_cfg* c) {
  if (c->bits < 2 || c->bits > 16) return ORC_VALUE;
  if (!(c->s_min > 0.0) || !(c->s_min < c->s_max)) return ORC_VALUE;
  if (!(c->eps > 0.0) || !(c->eps < c->s_min)) return ORC_VALUE;
  if (!(c->s_min_half > 0.0) || !(c->s_min_half < c->s_max)) return ORC_VALUE;
  return ORC_OK;
}

/* quant.hpp:45 */
int32_t orc_q_max(const orc_cfg* c) { return (1 << (c->bits - 1)) - 1; }

static double lower_bound(const orc_cfg* c, int half) {
  return half ? c->s_min_half : c->s_min; /* quant.hpp:47 */
}

/* ----------------------------------------------------------- scale math */

/* quant.hpp:71-75: log(1+e^x), large-x branch to stay finite. */
double orc_softplus(double x) {
  if (x > 30.0) return x + log1p(exp(-x));
  return log1p(exp(x));
}

/* quant.hpp:77-84: branch on the sign so exp never overflows. */
double orc_sigmoid(double x) {
  if (x < 0.0) {
    const double e = exp(x);
    return e / (1.0 + e);
  }
  return 1.0 / (1.0 + exp(-x));
}

/* quant.hpp:87-91 */
int orc_softplus_inv(double y, double* out) {
  if (y <= 0.0 || y != y) return ORC_VALUE;
  *out = (y > 30.0) ? y : log(expm1(y));
  return ORC_OK;
}

/* quant.hpp:95-101: min(max(softplus+eps, lo), s_max) in double. */
int orc_resolve_scale(double log_s, const orc_cfg* c, int half, double* out) {
  if (!isfinite(log_s)) return ORC_NONFINITE;
  const double raw = orc_softplus(log_s) + c->eps;
  const double lo = lower_bound(c, half);
  double s = raw < lo ? lo : raw;   /* std::max(raw, lo) */
  s = c->s_max < s ? c->s_max : s;  /* std::min(s, s_max) */
  *out = s;
  return ORC_OK;
}

/* ----------------------------------------------------------- binary16 */

/* half.hpp:17-42: RNE to binary16 bits; exponents past the half range
 * (including inf/NaN) pin to the largest finite code 0x7bff. */
uint16_t orc_f32_to_f16_bits(float v) {
  uint32_t u;
  memcpy(&u, &v, sizeof u);
  const uint16_t sign = (uint16_t)((u >> 16) & 0x8000u);
  const int32_t e = (int32_t)((u >> 23) & 0xffu) - 112; /* rebias 127 -> 15 */
  const uint32_t m = u & 0x7fffffu;
  if (e >= 31) return (uint16_t)(sign | 0x7bffu);
  if (e >= 1) {
    /* keep 10 mantissa bits, RNE on the 13 dropped ones; a carry may
     * legitimately ripple into the exponent field */
    uint32_t h = ((uint32_t)e << 10) | (m >> 13);
    const uint32_t drop = m & 0x1fffu;
    if (drop > 0x1000u || (drop == 0x1000u && (h & 1u))) h += 1u;
    return (uint16_t)(sign | h);
  }
  if (e < -10) return sign; /* below half the smallest subnormal */
  {
    const uint32_t full = m | 0x800000u; /* implicit bit */
    const uint32_t sh = (uint32_t)(14 - e); /* 14..24 */
    uint32_t h = full >> sh;
    const uint32_t drop = full & ((1u << sh) - 1u);
    const uint32_t mid = 1u << (sh - 1u);
    if (drop > mid || (drop == mid && (h & 1u))) h += 1u;
    return (uint16_t)(sign | h);
  }
}

/* half.hpp:44-68, restated arithmetically: subnormal m*2^-24, normal
 * (1024+m)*2^(e-25); all values exact in float. */
float orc_f16_bits_to_f32(uint16_t h) {
  const int neg = (h & 0x8000u) != 0;
  const int e = (h >> 10) & 0x1f;
  const int m = h & 0x3ff;
  float mag;
  if (e == 0) {
    mag = ldexpf((float)m, -24);
  } else if (e == 31) {
    /* inf / NaN: keep the payload bits (half.hpp:62-63) */
    const uint32_t u = 0x7f800000u | ((uint32_t)m << 13);
    memcpy(&mag, &u, sizeof mag);
  } else {
    mag = ldexpf((float)(1024 + m), e - 25);
  }
  return neg ? -mag : mag;
}

/* half.hpp:72-82 */
float orc_round_to_half(float v, int* saturated) {
  if (v > 65504.0f) {
    if (saturated) *saturated = 1;
    return 65504.0f;
  }
  if (v < -65504.0f) {
    if (saturated) *saturated = 1;
    return -65504.0f;
  }
  return orc_f16_bits_to_f32(orc_f32_to_f16_bits(v));
}

/* ------------------------------------------------------------ scalar FQ */

/* quant.hpp:114-121: float32 divide, NaN-propagating clip
 * (std::max/std::min are compare-selects), nearbyintf under the default
 * round-to-nearest-even mode, multiply s * r. */
float orc_fq_value(float x, float s, float q) {
  float z = x / s;
  z = (z < -q) ? -q : z; /* std::max(z, -q) */
  z = (q < z) ? q : z;   /* std::min(z, q)  */
  const float r = nearbyintf(z);
  return s * r;
}

/* ------------------------------------------------------ pairwise tree */

/* tensor.hpp:100-109: n <= 8 left fold in double, else split at n/2. */
double orc_pairwise_sum(const double* p, int64_t n) {
  if (n <= 8) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += p[i];
    return acc;
  }
  const int64_t h = n / 2;
  const double left = orc_pairwise_sum(p, h);
  const double right = orc_pairwise_sum(p + h, n - h);
  return left + right;
}

/* ---------------------------------------------------------- tensor ops */

static int check_positive(const double* s, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!(s[i] > 0.0)) return ORC_VALUE; /* quant.hpp:124-129 */
  return ORC_OK;
}

/* quant.hpp:136-146 (channels == 1) and :150-170 (axis-0 per-channel). */
int orc_fake_quantize(const float* x, float* y, int64_t outer, int64_t channels,
                      int64_t inner, const double* s, const orc_cfg* c,
                      int half) {
  int st = check_positive(s, channels);
  if (st) return st;
  const float q = (float)orc_q_max(c);
  int nonfinite = 0;
  for (int64_t o = 0; o < outer; ++o) {
    for (int64_t ch = 0; ch < channels; ++ch) {
      const float sf = (float)s[ch];
      const int64_t base = (o * channels + ch) * inner;
      for (int64_t i = 0; i < inner; ++i) {
        float v = orc_fq_value(x[base + i], sf, q);
        if (half) {
          /* demote_half (tensor.hpp:159-170) throws on non-finite; we
           * report it and store what round_to_half would */
          if (!isfinite(v)) nonfinite = 1;
          v = orc_round_to_half(v, NULL);
        }
        y[base + i] = v;
      }
    }
  }
  return nonfinite ? ORC_NONFINITE : ORC_OK;
}

/* exec.hpp:276-342: four whole-tensor sweeps with materialized float
 * temporaries; identical bits to the fused sweep because storing a float is
 * exact (quant.hpp:111-113). tmp3 holds 3*numel floats. */
int orc_fake_quantize_perop(const float* x, float* y, int64_t outer,
                            int64_t channels, int64_t inner, const double* s,
                            const orc_cfg* c, int half, float* tmp3) {
  int st = check_positive(s, channels);
  if (st) return st;
  const int64_t n = outer * channels * inner;
  const float q = (float)orc_q_max(c);
  float* t1 = tmp3;
  float* t2 = tmp3 + n;
  float* t3 = tmp3 + 2 * n;
#define ORC_SCALE_OF(i) ((float)s[((i) / inner) % channels])
  for (int64_t i = 0; i < n; ++i) t1[i] = x[i] / ORC_SCALE_OF(i);
  for (int64_t i = 0; i < n; ++i) {
    float z = t1[i];
    z = (z < -q) ? -q : z;
    t2[i] = (q < z) ? q : z;
  }
  for (int64_t i = 0; i < n; ++i) t3[i] = nearbyintf(t2[i]);
  int nonfinite = 0;
  for (int64_t i = 0; i < n; ++i) {
    float v = ORC_SCALE_OF(i) * t3[i];
    if (half) {
      if (!isfinite(v)) nonfinite = 1;
      v = orc_round_to_half(v, NULL);
    }
    y[i] = v;
  }
#undef ORC_SCALE_OF
  return nonfinite ? ORC_NONFINITE : ORC_OK;
}

/* quant.hpp:174-207: static_cast<int8_t>(nearbyintf(clip(x/s))). The
 * reference's float->int8 conversion of NaN goes through a 32-bit
 * truncation (x86 cvttss2si -> 0x80000000) whose low byte is 0. */
int orc_int8_codes(const float* x, int8_t* codes, int64_t outer,
                   int64_t channels, int64_t inner, const double* s,
                   const orc_cfg* c) {
  int st = check_positive(s, channels);
  if (st) return st;
  const float q = (float)orc_q_max(c);
  for (int64_t o = 0; o < outer; ++o) {
    for (int64_t ch = 0; ch < channels; ++ch) {
      const float sf = (float)s[ch];
      const int64_t base = (o * channels + ch) * inner;
      for (int64_t i = 0; i < inner; ++i) {
        float z = x[base + i] / sf;
        z = (z < -q) ? -q : z;
        z = (q < z) ? q : z;
        const float r = nearbyintf(z);
        const int32_t w = (r == r) ? (int32_t)r : 0;
        codes[base + i] = (int8_t)(uint8_t)(uint32_t)w;
      }
    }
  }
  return ORC_OK;
}

/* quant.hpp:217-228: per element, in double. */
static void grad_terms(double x, double s, double q, double* mask,
                       double* d_ds) {
  const double z = x / s;
  if (fabs(z) <= q) {
    *mask = 1.0;
    *d_ds = nearbyint(z) - z;
  } else {
    *mask = 0.0;
    *d_ds = (z > 0.0) ? q : -q;
  }
}

/* quant.hpp:233-294 generalized to [outer, channels, inner]: each row (o,c)
 * is one reference call's reduction (pairwise tree over the row, times the
 * clamp-gated sigmoid chain), accumulated over o in order. */
int orc_fq_backward(const float* x, const float* up, float* dx, int64_t outer,
                    int64_t channels, int64_t inner, const double* log_s,
                    const orc_cfg* c, int half, double* d_log_s,
                    int accumulate) {
  const double q = (double)orc_q_max(c);
  double* terms = (double*)malloc(sizeof(double) * (size_t)(inner > 0 ? inner : 1));
  if (!terms) return ORC_VALUE;
  for (int64_t ch = 0; ch < channels; ++ch) {
    double s;
    const int st = orc_resolve_scale(log_s[ch], c, half, &s);
    if (st) {
      free(terms);
      return st;
    }
    const double raw = orc_softplus(log_s[ch]) + c->eps;
    const int clamped = !(raw > lower_bound(c, half) && raw < c->s_max);
    const double chain = clamped ? 0.0 : orc_sigmoid(log_s[ch]);
    double acc = accumulate ? d_log_s[ch] : 0.0;
    for (int64_t o = 0; o < outer; ++o) {
      const int64_t base = (o * channels + ch) * inner;
      for (int64_t i = 0; i < inner; ++i) {
        double mask, d_ds;
        grad_terms((double)x[base + i], s, q, &mask, &d_ds);
        if (dx) dx[base + i] = (float)(mask * (double)up[base + i]);
        terms[i] = d_ds * (double)up[base + i];
      }
      const double r = orc_pairwise_sum(terms, inner) * chain;
      acc = (o == 0 && !accumulate) ? r : acc + r;
    }
    if (outer > 0) d_log_s[ch] = acc;
  }
  free(terms);
  return ORC_OK;
}

/* The same with the per-channel scale and chain factor given directly
 * (quant.hpp:281-292 after resolve_scale): reaches scales no log scale
 * resolves to (e.g. below 2^-100, the device's exact slow path). */
int orc_fq_backward_s(const float* x, const float* up, float* dx, int64_t outer,
                      int64_t channels, int64_t inner, const double* s,
                      const double* chain, double q, double* d_log_s) {
  double* terms = (double*)malloc(sizeof(double) * (size_t)(inner > 0 ? inner : 1));
  if (!terms) return ORC_VALUE;
  for (int64_t ch = 0; ch < channels; ++ch) {
    double acc = 0.0;
    for (int64_t o = 0; o < outer; ++o) {
      const int64_t base = (o * channels + ch) * inner;
      for (int64_t i = 0; i < inner; ++i) {
        double mask, d_ds;
        grad_terms((double)x[base + i], s[ch], q, &mask, &d_ds);
        if (dx) dx[base + i] = (float)(mask * (double)up[base + i]);
        terms[i] = d_ds * (double)up[base + i];
      }
      const double r = orc_pairwise_sum(terms, inner) * chain[ch];
      acc = (o == 0) ? r : acc + r;
    }
    if (outer > 0) d_log_s[ch] = acc;
  }
  free(terms);
  return ORC_OK;
}

float orc_gelu(float x) { return qfb_p_gelu(x); }

/* exec.hpp:438-451: v = maybe_half(act(add(a, b))) feeding the fused
 * activation sweeps of the consumers (exec.hpp:353-361). */
int orc_fq_chain(const float* a, const float* b, float* preact, float* y0,
                 float* y1, const double* s0, const double* s1,
                 int64_t outer, int64_t channels, int64_t inner, int act,
                 int half, const orc_cfg* c) {
  if (s0 && check_positive(s0, channels)) return ORC_VALUE;
  if (s1 && check_positive(s1, channels)) return ORC_VALUE;
  const float q = (float)orc_q_max(c);
  int nonfinite = 0;
  for (int64_t o = 0; o < outer; ++o) {
    for (int64_t ch = 0; ch < channels; ++ch) {
      const int64_t base = (o * channels + ch) * inner;
      for (int64_t i = 0; i < inner; ++i) {
        float v = a[base + i];
        if (b) v = v + b[base + i];                /* tensor.hpp:126-134 */
        if (act == 1) v = v > 0.0f ? v : 0.0f;     /* tensor.hpp:147-151 */
        else if (act == 2) v = qfb_p_gelu(v);
        if (half) {
          if (!isfinite(v)) nonfinite = 1;         /* tensor.hpp:160 */
          v = orc_round_to_half(v, NULL);
        }
        if (preact) preact[base + i] = v;
        if (y0) {
          float r = orc_fq_value(v, (float)s0[ch], q);
          if (half) r = orc_round_to_half(r, NULL); /* exec.hpp:357 */
          y0[base + i] = r;
        }
        if (y1) {
          float r = orc_fq_value(v, (float)s1[ch], q);
          if (half) r = orc_round_to_half(r, NULL);
          y1[base + i] = r;
        }
      }
    }
  }
  return nonfinite ? ORC_NONFINITE : ORC_OK;
}

/* ------------------------------------------------------------------ rng */

/* rng.hpp:15-21 splitmix64 finalizer. */
static uint64_t smix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* rng.hpp:29-32 */
uint64_t orc_rng_word(uint64_t seed, uint64_t stream, uint64_t index) {
  return smix(smix(seed ^ 0x243f6a8885a308d3ull) ^
              smix(stream * 0x9e3779b97f4a7c15ull + index));
}

/* rng.hpp:35-37: top 53 bits scaled by 2^-53. */
double orc_rng_uniform(uint64_t seed, uint64_t stream, uint64_t index) {
  return (double)(orc_rng_word(seed, stream, index) >> 11) * 0x1.0p-53;
}

/* rng.hpp:46-50: Irwin-Hall, sum of 12 uniforms minus 6. */
double orc_rng_normal(uint64_t seed, uint64_t stream, uint64_t index) {
  double acc = 0.0;
  for (uint64_t k = 0; k < 12; ++k)
    acc += orc_rng_uniform(seed, stream, index * 12 + k);
  return acc - 6.0;
}

void orc_fill_rng(float* out, int64_t n, uint64_t seed, uint64_t stream,
                  uint64_t offset, int kind, double lo, double hi, int half) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t idx = offset + (uint64_t)i;
    double v;
    if (kind == 0) {
      v = lo + (hi - lo) * orc_rng_uniform(seed, stream, idx); /* rng.hpp:40-42 */
    } else {
      v = lo * orc_rng_normal(seed, stream, idx);
    }
    float f = (float)v;
    if (half) f = orc_round_to_half(f, NULL);
    out[i] = f;
  }
}

/* ------------------------------------------- distillation loss (f3) */
/* pair_loss, distill.hpp:66-124, for one [c, hw] pair: out2 = {mse, mean
 * cosine}; d_s as the reference builds it (0.0f + float(2d/n), then += the
 * cosine term per location), finally scaled float(d * grad_scale) like the
 * trainer (distill.hpp:243-246). Returns 0, or 1 (ShapeError) for c < 1. */
int orc_distill_pair(const float* s, const float* t, int64_t c, int64_t hw, double lambda,
                     double grad_scale, float* d_s, double* out2) {
  if (c < 1 || hw < 1) return 1;
  const int64_t n = c * hw;
  double* sq = (double*)malloc(sizeof(double) * (size_t)n);
  double* cl = (double*)malloc(sizeof(double) * (size_t)hw);
  if (!sq || !cl) {
    free(sq);
    free(cl);
    return 2;
  }
  for (int64_t i = 0; i < n; ++i) {
    const double d = (double)s[i] - (double)t[i];
    sq[i] = d * d;
    d_s[i] = 0.0f + (float)(2.0 * d / (double)n);
  }
  out2[0] = orc_pairwise_sum(sq, n) / (double)n;
  const double w = lambda / (double)hw;
  for (int64_t p = 0; p < hw; ++p) {
    double dot = 0.0, na2 = 0.0, nb2 = 0.0;
    for (int64_t ch = 0; ch < c; ++ch) {
      const double a = s[ch * hw + p], b = t[ch * hw + p];
      dot += a * b;
      na2 += a * a;
      nb2 += b * b;
    }
    if (na2 == 0.0 || nb2 == 0.0) {
      cl[p] = 0.0;
      continue;
    }
    const double nrm = sqrt(na2 * nb2);
    const double cosv = dot / nrm;
    cl[p] = cosv;
    for (int64_t ch = 0; ch < c; ++ch) {
      const double a = s[ch * hw + p], b = t[ch * hw + p];
      d_s[ch * hw + p] += (float)(-w * (b / nrm - cosv * a / na2));
    }
  }
  out2[1] = orc_pairwise_sum(cl, hw) / (double)hw;
  for (int64_t i = 0; i < n; ++i) d_s[i] = (float)((double)d_s[i] * grad_scale);
  free(sq);
  free(cl);
  return 0;
}

/* Adam over the flattened scales, distill.hpp:264-279; returns 1 and leaves
 * everything unchanged when a gradient is non-finite (distill.hpp:254-258). */
int orc_adam(double* p, double* m, double* v, const double* g, int64_t n, double b1, double b2,
             double lr, double eps, int64_t t) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(g[i])) return 1;
  const double bc1 = 1.0 - pow(b1, (double)t);
  const double bc2 = 1.0 - pow(b2, (double)t);
  for (int64_t k = 0; k < n; ++k) {
    m[k] = b1 * m[k] + (1.0 - b1) * g[k];
    v[k] = b2 * v[k] + (1.0 - b2) * g[k] * g[k];
    const double mhat = m[k] / bc1;
    const double vhat = v[k] / bc2;
    p[k] -= lr * mhat / (sqrt(vhat) + eps);
  }
  return 0;
}
