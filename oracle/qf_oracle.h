/*
 * qf_oracle.h — CPU oracle for the fused fake-quant path.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C restatement of the
 * reference algorithm (quantfuse, /root/reference/proj/include/quantfuse)
 * used as the parity checker by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py. The product (libqfb.so) never links, loads
 * or calls it.
 *
 * Parity pinning: tests/test_oracle_vs_ref.py checks every function here
 * bitwise against the reference headers compiled from their own sources
 * (oracle/_ref/libqfref.so, recipe oracle/Makefile) and against the
 * committed golden vectors in tests/golden/ generated from that build.
 *
 * Config struct layout == qfb_quant_config (include/qfb.h).
 */
#ifndef QF_ORACLE_H_
#define QF_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_cfg {
  int32_t bits;
  int32_t reserved;
  double s_min, s_min_half, s_max, eps;
} orc_cfg;

enum { ORC_OK = 0, ORC_SHAPE = 1, ORC_VALUE = 2, ORC_NONFINITE = 4 };

/* quant.hpp:35-61 */
void orc_cfg_default(orc_cfg* c);
int orc_cfg_validate(const orc_cfg* c);
int32_t orc_q_max(const orc_cfg* c);

/* quant.hpp:71-109 */
double orc_softplus(double x);
double orc_sigmoid(double x);
int orc_softplus_inv(double y, double* out);
int orc_resolve_scale(double log_s, const orc_cfg* c, int half, double* out);

/* half.hpp:17-82 */
uint16_t orc_f32_to_f16_bits(float v);
float orc_f16_bits_to_f32(uint16_t h);
float orc_round_to_half(float v, int* saturated);

/* quant.hpp:114-121 */
float orc_fq_value(float x, float s, float q);

/* tensor.hpp:100-109 */
double orc_pairwise_sum(const double* p, int64_t n);

/* quant.hpp:136-170 over the [outer, channels, inner] view. half != 0:
 * EmulatedHalf input, result demoted (tensor.hpp:159-170): returns
 * ORC_NONFINITE (after writing) if any result is non-finite. Non-finite
 * results under half are written as round_to_half would (+-65504). */
int orc_fake_quantize(const float* x, float* y, int64_t outer, int64_t channels,
                      int64_t inner, const double* s, const orc_cfg* c, int half);

/* Per-operator form: divide, clip, round, multiply as four sweeps with
 * materialized temporaries (exec.hpp:276-342). */
int orc_fake_quantize_perop(const float* x, float* y, int64_t outer,
                            int64_t channels, int64_t inner, const double* s,
                            const orc_cfg* c, int half, float* tmp3);

/* quant.hpp:174-207; NaN -> 0. */
int orc_int8_codes(const float* x, int8_t* codes, int64_t outer,
                   int64_t channels, int64_t inner, const double* s,
                   const orc_cfg* c);

/* quant.hpp:217-294 + accumulation of frontend.hpp:222-228 (see qfb.h). */
int orc_fq_backward(const float* x, const float* up, float* dx, int64_t outer,
                    int64_t channels, int64_t inner, const double* log_s,
                    const orc_cfg* c, int half, double* d_log_s, int accumulate);
int orc_fq_backward_s(const float* x, const float* up, float* dx, int64_t outer,
                      int64_t channels, int64_t inner, const double* s,
                      const double* chain, double q, double* d_log_s);

/* Fused chain (exec.hpp:438-451 + :353-361). act: 0 none, 1 relu, 2 gelu.
 * s0/s1: double scales (cast to float), NULL when unused. */
int orc_fq_chain(const float* a, const float* b, float* preact, float* y0,
                 float* y1, const double* s0, const double* s1,
                 int64_t outer, int64_t channels, int64_t inner, int act,
                 int half, const orc_cfg* c);

float orc_gelu(float x);

/* rng.hpp:15-50 */
uint64_t orc_rng_word(uint64_t seed, uint64_t stream, uint64_t index);
double orc_rng_uniform(uint64_t seed, uint64_t stream, uint64_t index);
double orc_rng_normal(uint64_t seed, uint64_t stream, uint64_t index);
/* kind 0: lo + (hi-lo)*uniform; kind 1: lo * normal. Rounded to float
 * (half != 0: then to the binary16 grid). */
void orc_fill_rng(float* out, int64_t n, uint64_t seed, uint64_t stream,
                  uint64_t offset, int kind, double lo, double hi, int half);

/* distill.hpp:66-124 (one pair) and :264-279 (Adam) */
int orc_distill_pair(const float* s, const float* t, int64_t c, int64_t hw, double lambda,
                     double grad_scale, float* d_s, double* out2);
int orc_adam(double* p, double* m, double* v, const double* g, int64_t n, double b1, double b2,
             double lr, double eps, int64_t t);

#ifdef __cplusplus
}
#endif
#endif
