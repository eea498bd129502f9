/*
 * qfb_portable.h — arithmetic that must give identical bits on the host
 * (gcc, x86-64, -ffp-contract=off) and on the device (nvcc, sm_100a).
 *
 * Only IEEE-754 basic operations with round-to-nearest-even are used (add,
 * mul, fma), each spelled through a macro that maps to the correctly
 * rounded intrinsic on the device and to the plain operator / libm fmaf
 * (correctly rounded) on the host. No libm transcendental is called, so the result
 * does not depend on either side's libm.
 *
 * GELU: the reference has no GELU (parity unpinned). This
 * header DEFINES the GELU of the fused chain (the erf form x * Phi(x)
 * with Phi from a polynomial; see qfb_p_gelu), and the
 * CPU oracle includes this same header, so oracle and kernel agree bitwise
 * by construction. It is the only code shared by oracle and product.
 */
#ifndef QFB_PORTABLE_H_
#define QFB_PORTABLE_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define QFB_HD __host__ __device__ __forceinline__
#else
#define QFB_HD static inline
#include <math.h>
#endif

#if defined(__CUDA_ARCH__)
#define QFB_P_ADD(a, b) __fadd_rn((a), (b))
#define QFB_P_MUL(a, b) __fmul_rn((a), (b))
#define QFB_P_FMA(a, b, c) __fmaf_rn((a), (b), (c))
#else
#define QFB_P_ADD(a, b) ((a) + (b))
#define QFB_P_MUL(a, b) ((a) * (b))
#define QFB_P_FMA(a, b, c) fmaf((a), (b), (c))
#endif

/* GELU(x) = x * Phi(x), Phi the standard normal CDF (the erf GELU):
 * Phi(x) = 0.5 + sign(x) * h(|x|), h(t) = 0.5 * erf(t / sqrt 2) on [0, 5]
 * as a degree-12 polynomial in u = 0.4 t - 1 (Chebyshev fit, float32
 * coefficients, Horner with FMAs); beyond |x| > 5, Phi is 1 or 0 exactly.
 * Within 2.1e-6 of the erf GELU. NaN passes through; +inf -> +inf,
 * -inf -> -0. FMAs, one multiply and one add: identical bits on both sides. */
/* The Horner coefficients of h, highest degree first (shared by the scalar
 * form below and the device's packed two-lane form). */
#define QFB_P_GELU_C0 0.010865055f
#define QFB_P_GELU_HORNER(STEP)                                                 \
  STEP(-0.013859635f) STEP(-0.041010167f) STEP(0.07832172f) STEP(0.025033878f) \
  STEP(-0.16348906f) STEP(0.13090801f) STEP(0.0655948f) STEP(-0.23270182f)     \
  STEP(0.23961057f) STEP(-0.13688436f) STEP(0.043821268f) STEP(0.49378976f)

/* x * Phi(x) from the polynomial, for -5 <= x <= 5 (qfb_p_gelu's middle
 * branch; the device's branch-free form selects around it). */
QFB_HD float qfb_p_gelu_core(float x) {
  const float t = x < 0.0f ? -x : x;
  const float u = QFB_P_FMA(t, 0.4f, -1.0f);
  float h = QFB_P_GELU_C0;
#define QFB_P_GELU_STEP(c) h = QFB_P_FMA(h, u, c);
  QFB_P_GELU_HORNER(QFB_P_GELU_STEP)
#undef QFB_P_GELU_STEP
  const float phi = QFB_P_ADD(0.5f, x < 0.0f ? -h : h);
  return QFB_P_MUL(x, phi);
}

QFB_HD float qfb_p_gelu(float x) {
  if (!(x == x)) return x;
  if (x > 5.0f) return x;
  if (x < -5.0f) return -0.0f;
  return qfb_p_gelu_core(x);
}

#endif /* QFB_PORTABLE_H_ */
