/*
 * qfb_portable.h — arithmetic that must give identical bits on the host
 * (gcc, x86-64, -ffp-contract=off) and on the device (nvcc, sm_100a).
 *
 * Only IEEE-754 basic operations with round-to-nearest-even are used (add,
 * mul, div, fma, rint), each spelled through a macro that maps to the
 * correctly rounded intrinsic on the device and to the plain operator /
 * libm fmaf on the host. No libm transcendental is called, so the result
 * does not depend on either side's libm.
 *
 * GELU: the reference has no GELU (parity unpinned). This
 * header DEFINES the GELU of the fused chain (tanh form,
 * 0.5*x*(1+tanh(sqrt(2/pi)*(x+0.044715*x^3))), evaluated as
 * x*(1/(1+e^{-2u})) with a portable exp), and the
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
#include <string.h>
#endif

#if defined(__CUDA_ARCH__)
#define QFB_P_ADD(a, b) __fadd_rn((a), (b))
#define QFB_P_MUL(a, b) __fmul_rn((a), (b))
#define QFB_P_DIV(a, b) __fdiv_rn((a), (b))
#define QFB_P_FMA(a, b, c) __fmaf_rn((a), (b), (c))
#define QFB_P_RINT(a) rintf(a)
#define QFB_P_RCP(a) __frcp_rn(a)
#define QFB_P_AS_FLOAT(u) __uint_as_float(u)
#define QFB_P_AS_UINT(f) __float_as_uint(f)
#else
#define QFB_P_ADD(a, b) ((a) + (b))
#define QFB_P_MUL(a, b) ((a) * (b))
#define QFB_P_DIV(a, b) ((a) / (b))
#define QFB_P_FMA(a, b, c) fmaf((a), (b), (c))
#define QFB_P_RINT(a) rintf(a)
#define QFB_P_RCP(a) (1.0f / (a))
QFB_HD float qfb_p_as_float_(uint32_t u) {
  float f;
  memcpy(&f, &u, sizeof f);
  return f;
}
QFB_HD uint32_t qfb_p_as_uint_(float f) {
  uint32_t u;
  memcpy(&u, &f, sizeof u);
  return u;
}
#define QFB_P_AS_FLOAT(u) qfb_p_as_float_(u)
#define QFB_P_AS_UINT(f) qfb_p_as_uint_(f)
#endif

/* 2^j for j in [-126, 127], built from the exponent field. */
QFB_HD float qfb_p_exp2i(int32_t j) {
  return QFB_P_AS_FLOAT((uint32_t)(j + 127) << 23);
}

/* tanh-form GELU, 0.5 x (1 + tanh(u)) with u = sqrt(2/pi) (x + 0.044715 x^3),
 * evaluated as the identical x * sigmoid(2u) = x * (1 / (1 + e^{-2u})).
 * e^t is computed for t = -2u clamped to [-30, 88] (below -30, 1 + e^t == 1
 * in float; above 88 the result is x * 0): magic-number rounding
 * k = RN(t / ln2) (1.5 * 2^23 added and subtracted), Cody-Waite reduction,
 * degree-5 Taylor/Horner on |r| <= ln2/2 (relative error < 3e-6) and one
 * exponent scaling 2^k, k in [-44, 127]. Then one correctly rounded
 * reciprocal and a multiply. NaN passes through; -inf -> -0. Within 2e-3 of
 * the erf GELU (tests/test_gpu_fwd.py::test_gelu_portable_bitwise). */
QFB_HD float qfb_p_gelu(float x) {
  if (!(x == x)) return x;
  if (x < -3.0e38f) return -0.0f;
  const float x3 = QFB_P_MUL(QFB_P_MUL(x, x), x);
  const float u = QFB_P_MUL(0.7978845834732055664f, QFB_P_FMA(0.044715f, x3, x));
  float t = QFB_P_MUL(-2.0f, u);
  if (t > 88.0f) return QFB_P_MUL(x, 0.0f);
  t = t < -30.0f ? -30.0f : t;
  const float m = QFB_P_ADD(QFB_P_MUL(t, 1.44269502162933349609375f), 12582912.0f);
  const float kf = QFB_P_ADD(m, -12582912.0f);
  const int32_t k = (int32_t)(QFB_P_AS_UINT(m) - 0x4B400000u);
  float r = QFB_P_FMA(kf, -0.693145751953125f, t);      /* ln2 hi (exact k*hi) */
  r = QFB_P_FMA(kf, -1.428606765330187045e-06f, r);     /* ln2 lo */
  float p = 8.33333377e-3f;                              /* 1/120 */
  p = QFB_P_FMA(p, r, 4.16666679e-2f);                   /* 1/24  */
  p = QFB_P_FMA(p, r, 1.66666672e-1f);                   /* 1/6   */
  p = QFB_P_FMA(p, r, 0.5f);
  p = QFB_P_FMA(p, r, 1.0f);
  p = QFB_P_FMA(p, r, 1.0f);
  const float e = QFB_P_MUL(p, qfb_p_exp2i(k));
  return QFB_P_MUL(x, QFB_P_RCP(QFB_P_ADD(1.0f, e)));
}

#endif /* QFB_PORTABLE_H_ */
