/*
 * qfb.h — C-ABI of the B200-native fused fake-quantization path ("qfb").
 *
 * This is the drop-in boundary for the DPVO-QAT++ accelerator path
 * (arxiv 2511.12653). Every entry point replaces one operator of the
 * reference library `quantfuse` (namespace qf, /root/reference/proj); the
 * reference interface each one replaces is cited as file:line (paths relative
 * to proj/include/quantfuse/).
 *
 * Conventions
 *  - Plain C types only: pointers, sizes, enums, POD structs. No torch types.
 *  - Every function returns qfb_status; on failure qfb_last_error() holds a
 *    thread-local message. Status codes mirror the reference exception
 *    taxonomy (errors.hpp:11-33, exec.hpp:51-53).
 *  - Device entry points (qfb_fq_*, qfb_int8_codes, qfb_fill_*) take DEVICE
 *    pointers, validate arguments on the host before anything is enqueued
 *    (validation-before-compute, as in quant.hpp:124-157), then enqueue
 *    asynchronously on the context's stream. They never allocate on the hot
 *    path except to grow the context workspace. Device-detected conditions
 *    (non-finite values where the reference throws NonFiniteError) are
 *    latched in the context and reported by qfb_ctx_sync().
 *  - Host entry points (*_host) mirror the reference's value-semantics API:
 *    host buffers in, host buffers out, synchronous, all copies inside.
 *  - Layout: every tensor is viewed as [outer, channels, inner] row-major.
 *    Element i uses scale index (i / inner) % channels. Per-tensor scale is
 *    channels == 1. The reference's per-channel axis-0 form
 *    (quant.hpp:150-170, [C_out, per]) is outer=1, channels=C_out,
 *    inner=per; a batch of CHW frames with per-channel activation scales is
 *    outer=frames, channels=C, inner=H*W.
 *  - A context is externally single-threaded (exec.hpp:180-181); distinct
 *    contexts may be used from distinct threads.
 */
#ifndef QFB_H_
#define QFB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QFB_VERSION_MAJOR 0
#define QFB_VERSION_MINOR 1

/* ---------------------------------------------------------------------- */
/* Status codes: errors.hpp:11-33 (ShapeError, ValueError, IoError,        */
/* NonFiniteError, InsufficientMatchesError) + exec.hpp:51 FusedPathError. */
/* ---------------------------------------------------------------------- */
typedef enum qfb_status {
  QFB_OK = 0,
  QFB_ERR_SHAPE = 1,          /* qf::ShapeError               errors.hpp:11 */
  QFB_ERR_VALUE = 2,          /* qf::ValueError               errors.hpp:16 */
  QFB_ERR_IO = 3,             /* qf::IoError                  errors.hpp:21 */
  QFB_ERR_NONFINITE = 4,      /* qf::NonFiniteError           errors.hpp:26 */
  QFB_ERR_INSUFFICIENT = 5,   /* qf::InsufficientMatchesError errors.hpp:31 */
  QFB_ERR_FUSED_PATH = 6,     /* qf::FusedPathError           exec.hpp:51   */
  QFB_ERR_CUDA = 7,           /* CUDA runtime / launch failure              */
  QFB_ERR_NCCL = 8,           /* collective failure                         */
  QFB_ERR_UNSUPPORTED = 9     /* argument combination not supported         */
} qfb_status;

/* Thread-local message of the last failing call on this thread. */
const char* qfb_last_error(void);
const char* qfb_status_name(qfb_status s);
/* Library build string (arch, version). */
const char* qfb_build_info(void);

/* Storage type of device tensors. */
typedef enum qfb_dtype {
  QFB_F32 = 0, /* float32 storage                                        */
  QFB_F16 = 1  /* IEEE binary16 storage (the reference's EmulatedHalf     */
               /* values are exactly these, tensor.hpp:25, half.hpp:1-5) */
} qfb_dtype;

/* qf::Precision (tensor.hpp:23). Selects the activation scale lower bound
 * (quant.hpp:45-47) and, for float32 storage, whether results are re-rounded
 * onto the binary16 grid (quant.hpp:141-143). */
typedef enum qfb_precision {
  QFB_PREC_FULL = 0,
  QFB_PREC_HALF = 1
} qfb_precision;

/* Kernel flags. */
#define QFB_FLAG_HALF_GRID 0x1u /* f32 storage: round outputs to binary16 */
                                /* grid (round_to_half, half.hpp:72-82)   */
#define QFB_FLAG_STREAMING 0x2u /* evict-first loads/stores (data >> L2)  */
#define QFB_FLAG_INT8_OUT  0x4u /* qfb_fq_fwd_multi: every output y[k] of */
                                /* the entry receives the int8 codes      */
                                /* (int8_codes, quant.hpp:174-207; 1 byte */
                                /* per element) instead of FQ values      */

/* ---------------------------------------------------------------------- */
/* Quantization config: qf::QuantConfig (quant.hpp:35-61).                */
/* ---------------------------------------------------------------------- */
typedef struct qfb_quant_config {
  int32_t bits;       /* default 8 -> q_max 127                          */
  int32_t reserved;
  double s_min;       /* 1e-6, Full path lower clamp                     */
  double s_min_half;  /* 1e-4, FP16 path lower clamp                     */
  double s_max;       /* 64                                              */
  double eps;         /* 1e-8                                            */
} qfb_quant_config;

void qfb_quant_config_default(qfb_quant_config* cfg);          /* quant.hpp:35-43 */
qfb_status qfb_quant_config_validate(const qfb_quant_config*); /* quant.hpp:49-60 */
int32_t qfb_q_max(const qfb_quant_config* cfg);                /* quant.hpp:45    */

/* ---------------------------------------------------------------------- */
/* Host scale math — computed with the host libm so the resolved scales are */
/* bit-identical to the reference on the same machine.                     */
/* ---------------------------------------------------------------------- */
double qfb_softplus(double x);                           /* quant.hpp:71-75 */
double qfb_sigmoid(double x);                            /* quant.hpp:77-84 */
qfb_status qfb_softplus_inv(double y, double* out);      /* quant.hpp:87-91 */
/* s = clip(softplus(log_s)+eps, s_min_for(prec), s_max); quant.hpp:95-109.
 * Non-finite log_s -> QFB_ERR_NONFINITE. */
qfb_status qfb_resolve_scales(const double* log_s, int64_t n,
                              const qfb_quant_config* cfg, qfb_precision prec,
                              double* s_out);
/* Backward factors per scale: s (double, quant.hpp:241/281) and
 * chain = clamped ? 0 : sigmoid(log_s) (quant.hpp:242-244, 282-284). */
qfb_status qfb_scale_grad_factors(const double* log_s, int64_t n,
                                  const qfb_quant_config* cfg,
                                  qfb_precision prec, double* s_out,
                                  double* chain_out);
/* Forward scale contract: reject s <= 0 (ValueError, quant.hpp:124-129) and
 * cast to float (quant.hpp:138, 162; exec.hpp:250-254). */
qfb_status qfb_cast_scales_f32(const double* s, int64_t n, float* out);

/* ---------------------------------------------------------------------- */
/* Context: one per (device, stream); owns the reduction workspace and the */
/* device status latch.                                                     */
/* ---------------------------------------------------------------------- */
typedef struct qfb_ctx qfb_ctx;

/* stream: a cudaStream_t (NULL = the legacy default stream). */
qfb_status qfb_ctx_create(int32_t device, void* stream, qfb_ctx** out);
qfb_status qfb_ctx_destroy(qfb_ctx* ctx);
qfb_status qfb_ctx_set_stream(qfb_ctx* ctx, void* stream);
/* Context options. QFB_OPT_BWD_HALF_FP32 (value 0/1, default 0): binary16
 * storage only — the STE/LSQ backward computes its scale-gradient terms in
 * float32 instead of the reference's binary64 (quant.hpp:217-228). d_input
 * stays bit-identical (the clip mask is decided exactly); d_log_s agrees
 * with the reference within the FP16 tolerance (rel 1e-2; measured ~1e-6,
 * DESIGN.md §2) instead of bitwise. Off: every result is bitwise. */
#define QFB_OPT_BWD_HALF_FP32 1
/* QFB_OPT_MAIN_PASS_EVENT (value: a cudaEvent_t cast to int64, 0 = off):
 * profiling hook — each backward call records the event on the context
 * stream between its main pass and its finisher kernel, so a caller can
 * time the main pass alone with events (bench.py's roofline). */
#define QFB_OPT_MAIN_PASS_EVENT 2
/* QFB_OPT_BWD_ASYNC_FINISH (value 0/1, default 0): the backward's finisher
 * (the per-row tree of tile partials -> d_log_s) runs on a context-owned
 * side stream, forked after the main pass, so the caller's next kernels
 * (e.g. the next frame's forward) overlap it. d_log_s is then complete
 * only after a JOIN point in the context stream's order: the next
 * backward call on this context (which reuses the partials workspace),
 * qfb_ctx_join, or qfb_ctx_sync. Capturable (event fork/join); a capture
 * must qfb_ctx_join before it ends. */
#define QFB_OPT_BWD_ASYNC_FINISH 3
qfb_status qfb_ctx_set_option(qfb_ctx* ctx, int32_t option, int64_t value);
/* Make the context stream wait for any work the context forked to its side
 * stream (QFB_OPT_BWD_ASYNC_FINISH); no-op otherwise. Stream-ordered,
 * capturable. */
qfb_status qfb_ctx_join(qfb_ctx* ctx);
void* qfb_ctx_stream(qfb_ctx* ctx);
int32_t qfb_ctx_sm_count(qfb_ctx* ctx);
/* Synchronize the stream; report (and clear) latched device conditions.
 * Returns QFB_ERR_NONFINITE if a kernel saw a non-finite value where the
 * reference throws (demote_half, tensor.hpp:160). */
qfb_status qfb_ctx_sync(qfb_ctx* ctx);
/* Number of kernels this context has launched (for launch accounting). */
int64_t qfb_ctx_launch_count(qfb_ctx* ctx);

/* ---------------------------------------------------------------------- */
/* Device operators (async on the context stream, device pointers).        */
/* ---------------------------------------------------------------------- */

/* Fake-quant forward, y = s*rint(clip(x/s, -q, q)) in float32 with IEEE
 * division, round-half-even, NaN-propagating clip and signed zero.
 * Replaces qf::fake_quantize per-tensor (quant.hpp:136-146) and per-channel
 * (quant.hpp:150-170), scalar kernel quant.hpp:114-121.
 * scale: device float[channels] (already cast, see qfb_cast_scales_f32).
 * x == y (in place) is allowed. */
qfb_status qfb_fq_fwd(qfb_ctx* ctx, qfb_dtype dtype, const void* x, void* y,
                      int64_t outer, int64_t channels, int64_t inner,
                      const float* scale, int32_t q_max, uint32_t flags);

/* Integer image: codes = (int8)rint(clip(x/s)). qf::int8_codes
 * (quant.hpp:174-207). NaN -> 0. */
qfb_status qfb_int8_codes(qfb_ctx* ctx, qfb_dtype dtype, const void* x,
                          int8_t* codes, int64_t outer, int64_t channels,
                          int64_t inner, const float* scale, int32_t q_max);

/* STE/LSQ backward with the reference's fixed pairwise reduction tree
 * (tensor.hpp:100-109) reproduced exactly on the device.
 * Replaces qf::fake_quantize_backward per-tensor (quant.hpp:233-257) and
 * per-channel (quant.hpp:261-294).
 *  dx (nullable, frozen weights, frontend.hpp:221-225): mask * up.
 *  scale64 / chain: device double[channels] from qfb_scale_grad_factors.
 *  d_log_s: device double[channels]. Row (o,c) yields
 *    r[o][c] = pairwise_sum(d_ds * up over the row) * chain[c].
 *  accumulate == 0: d_log_s[c] = ((r[0][c] + r[1][c]) + ...)
 *  accumulate == 1: d_log_s[c] = ((d_log_s[c] + r[0][c]) + r[1][c]) + ...
 *    (the trainer's `g += grad` accumulation, frontend.hpp:222-228).
 *  accumulate == QFB_BWD_ROWS (2): one result per row, no fold:
 *    d_log_s[o * row_stride + c] = r[o][c] (row_stride = channels here,
 *    settable per entry in qfb_bwd_desc). The rows of frames sharded over
 *    GPUs are gathered and folded in frame order by
 *    qfb_gather_fold_scale_grads / qfb_fold_rows, which reproduces the
 *    single-process fold bit for bit. */
#define QFB_BWD_ROWS 2
qfb_status qfb_fq_bwd(qfb_ctx* ctx, qfb_dtype dtype, const void* x,
                      const void* up, void* dx, int64_t outer,
                      int64_t channels, int64_t inner, const double* scale64,
                      const double* chain, int32_t q_max, double* d_log_s,
                      int32_t accumulate);

/* Activation applied inside a fused chain. */
typedef enum qfb_act {
  QFB_ACT_NONE = 0,
  QFB_ACT_RELU = 1, /* v > 0 ? v : 0, tensor.hpp:147-151               */
  QFB_ACT_GELU = 2  /* portable tanh-GELU, include/qfb_portable.h      */
} qfb_act;

#define QFB_MAX_CHAIN_OUT 2

/* Fused quant->act->quant chain over one tensor (one HBM pass):
 *   v = a (+ b); v = act(v); if half: v = demote(v) (non-finite latched,
 *   tensor.hpp:159-170); preact = v (optional);
 *   y[k] = FQ(v, scale[k]) (+ half re-round) for k < n_out.
 * Semantics: the residual joins maybe_half(relu(add(a,b))) of
 * exec.hpp:438,443,447 followed by the next layers' fused activation
 * sweep exec.hpp:353-361, including multi-consumer points exec.hpp:440-451. */
typedef struct qfb_chain_desc {
  const void* a;
  const void* b;         /* nullable */
  void* preact;          /* nullable */
  void* y[QFB_MAX_CHAIN_OUT];
  const float* scale[QFB_MAX_CHAIN_OUT]; /* device float[channels] each */
  int64_t outer, channels, inner;
  int32_t n_out;         /* 0..2 */
  int32_t act;           /* qfb_act */
  int32_t dtype;         /* qfb_dtype */
  int32_t q_max;
  uint32_t flags;        /* QFB_FLAG_* */
  uint32_t reserved;
} qfb_chain_desc;

qfb_status qfb_fq_chain(qfb_ctx* ctx, const qfb_chain_desc* desc);

/* Batched launches: one kernel over a table of quant points (all the
 * activation quant points of a frame or window). The table is passed by
 * value in kernel parameters, so calls are CUDA-graph capturable. */
typedef struct qfb_fq_desc {
  const void* x;
  void* y[QFB_MAX_CHAIN_OUT];            /* y[1] used when n_out == 2 */
  const float* scale[QFB_MAX_CHAIN_OUT];
  int64_t outer, channels, inner;
  int32_t n_out;   /* 1 or 2 (multi-consumer quant point, one read of x) */
  int32_t q_max;
  uint32_t flags;
  uint32_t reserved;
} qfb_fq_desc;

qfb_status qfb_fq_fwd_multi(qfb_ctx* ctx, qfb_dtype dtype,
                            const qfb_fq_desc* table, int32_t n);

typedef struct qfb_bwd_desc {
  const void* x;
  const void* up;
  void* dx;                 /* nullable */
  const double* scale64;
  const double* chain;
  double* d_log_s;
  int64_t outer, channels, inner;
  int32_t q_max;
  int32_t accumulate;       /* 0, 1 or QFB_BWD_ROWS (see qfb_fq_bwd) */
  int64_t row_stride;       /* QFB_BWD_ROWS: doubles between rows (0: channels) */
} qfb_bwd_desc;

qfb_status qfb_fq_bwd_multi(qfb_ctx* ctx, qfb_dtype dtype,
                            const qfb_bwd_desc* table, int32_t n);
/* Size the context's backward workspace for `table` without launching, so
 * the first call may be made under stream capture (growth during a capture
 * is refused with QFB_ERR_UNSUPPORTED; buffers a captured graph references
 * are never freed before qfb_ctx_destroy). */
qfb_status qfb_fq_bwd_reserve(qfb_ctx* ctx, qfb_dtype dtype,
                              const qfb_bwd_desc* table, int32_t n);

qfb_status qfb_fq_chain_multi(qfb_ctx* ctx, const qfb_chain_desc* table,
                              int32_t n);

/* Device-side scale resolution (the paper's scale kernel):
 * CUDA libm, may differ from the host libm by <= 1-2 ulp in double.
 * Any output pointer may be NULL. Non-finite log_s is latched
 * (QFB_ERR_NONFINITE at qfb_ctx_sync). */
qfb_status qfb_resolve_scales_dev(qfb_ctx* ctx, const double* log_s,
                                  int64_t n, const qfb_quant_config* cfg,
                                  qfb_precision prec, float* s32,
                                  double* s64, double* chain);

/* Synthetic input generation on the device with the reference counter RNG
 * (rng.hpp:24-50), so host and device see identical bytes without H2D:
 * out[i] = (dtype)(lo + (hi - lo) * uniform(i))   (kind 0)
 * out[i] = (dtype)(scale * normal(i))              (kind 1; lo = scale)
 * with index i + index_offset. */
qfb_status qfb_fill_rng(qfb_ctx* ctx, qfb_dtype dtype, void* out, int64_t n,
                        uint64_t seed, uint64_t stream, uint64_t index_offset,
                        int32_t kind, double lo, double hi);

/* ---------------------------------------------------------------------- */
/* Per-operator plan (ablation + fused-path fallback), exec.hpp:276-342:   */
/* four sweeps divide -> clip -> round -> multiply with materialized       */
/* float temporaries (z, c, r), bit-identical to the fused sweep.          */
/* tmp: device float[3 * numel] scratch.                                   */
/* ---------------------------------------------------------------------- */
qfb_status qfb_fq_fwd_perop(qfb_ctx* ctx, qfb_dtype dtype, const void* x,
                            void* y, int64_t outer, int64_t channels,
                            int64_t inner, const float* scale, int32_t q_max,
                            uint32_t flags, float* tmp);

/* ---------------------------------------------------------------------- */
/* Host-level operators with reference value semantics (quant.hpp).        */
/* Float32 host buffers; prec == QFB_PREC_HALF means the input is an       */
/* EmulatedHalf tensor (values on the binary16 grid) and the output is     */
/* re-rounded onto that grid; a non-finite result -> QFB_ERR_NONFINITE as  */
/* demote_half would throw (tensor.hpp:160). Synchronous.                  */
/* ---------------------------------------------------------------------- */
/* s: host double[channels] (validated > 0 and cast to float). */
qfb_status qfb_fake_quantize_host(qfb_ctx* ctx, qfb_precision prec,
                                  const float* x, float* y, int64_t outer,
                                  int64_t channels, int64_t inner,
                                  const double* s,
                                  const qfb_quant_config* cfg);
qfb_status qfb_int8_codes_host(qfb_ctx* ctx, const float* x, int8_t* codes,
                               int64_t outer, int64_t channels, int64_t inner,
                               const double* s, const qfb_quant_config* cfg);
/* log_s: host double[channels]; d_log_s: host double[channels] (written,
 * or accumulated into when accumulate != 0); dx nullable. */
qfb_status qfb_fake_quantize_backward_host(
    qfb_ctx* ctx, qfb_precision prec, const float* x, const float* up,
    float* dx, int64_t outer, int64_t channels, int64_t inner,
    const double* log_s, const qfb_quant_config* cfg, double* d_log_s,
    int32_t accumulate);

/* ---------------------------------------------------------------------- */
/* Execution plan: the quant part of qf::run_quant_conv (exec.hpp:222-405) */
/* — scale pass, activation FQ, weight FQ — under a PerOperator (four      */
/* materialized sweeps each) or Fused (one sweep each) plan, with the      */
/* fused-path fault hook and fallback, the frozen-weight cache and the     */
/* modeled pass/byte counters (exec.hpp:199-216). The convolution itself   */
/* stays with the caller (cuDNN).                            */
/* ---------------------------------------------------------------------- */
typedef enum qfb_exec_mode { QFB_MODE_PER_OPERATOR = 0, QFB_MODE_FUSED = 1 } qfb_exec_mode; /* exec.hpp:43 */
typedef enum qfb_precision_policy {
  QFB_POLICY_FULL_ONLY = 0, QFB_POLICY_HALF_ACTIVATIONS = 1                              /* exec.hpp:44 */
} qfb_precision_policy;

typedef struct qfb_exec_plan {   /* qf::ExecutionPlan, exec.hpp:55-65 */
  int32_t mode;                  /* qfb_exec_mode */
  int32_t policy;                /* qfb_precision_policy */
  int32_t fallback_enabled;      /* fused failure -> per-operator rerun */
  int32_t cache_weights;         /* quantize frozen weights once per plan */
  int32_t fault_inject_layer;    /* test hook: fused path fails at this layer (-1 off) */
  int32_t reserved;
} qfb_exec_plan;

typedef struct qfb_exec_trace {  /* qf::ExecutionTrace counters, exec.hpp:75-98 */
  int64_t pass_count;            /* modeled sweeps (scale + quant; conv is the caller's) */
  int64_t bytes_read;
  int64_t bytes_written;
  int64_t launches;              /* device kernels actually launched */
  int64_t peak_scratch_bytes;    /* per-operator temporaries (allocated peak) */
  int32_t fell_back;
  int32_t layers;
} qfb_exec_trace;

/* One layer's quantization state (qf::ConvLayer quant fields, model.hpp). */
typedef struct qfb_quant_layer {
  int32_t index;                 /* roster index: fault hook + cache key */
  int32_t reserved;
  const float* weight;           /* device [c_out, per], float32 */
  int64_t c_out, per;
  const double* log_w;           /* host [c_out] log weight scales */
  double log_a;                  /* log activation scale */
} qfb_quant_layer;

typedef struct qfb_exec qfb_exec;
qfb_status qfb_exec_create(qfb_ctx* ctx, const qfb_exec_plan* plan, qfb_exec** out);
qfb_status qfb_exec_destroy(qfb_exec* ex);
/* Quantize one layer's activation x (device, dtype, [outer, channels,
 * inner] viewed per-tensor as in the reference) into qa (device, same
 * dtype) and its weights into *qw (device float[c_out*per]; points at the
 * plan's cache when cache_weights, else at qw_buf which the caller owns).
 * Returns QFB_ERR_FUSED_PATH when the injected fault fires without
 * fallback. */
qfb_status qfb_exec_quant_layer(qfb_exec* ex, const qfb_quant_layer* layer,
                                const qfb_quant_config* cfg, qfb_dtype dtype,
                                const void* x, int64_t n_act, void* qa,
                                float* qw_buf, const float** qw);
qfb_status qfb_exec_trace_get(const qfb_exec* ex, qfb_exec_trace* out);
qfb_status qfb_exec_trace_reset(qfb_exec* ex);
/* The modeled counter increments of one layer, exec.hpp:203-214 byte rules
 * (host only, no GPU): for the schedule-walker tests (test_exec.cpp:31-92). */
qfb_status qfb_exec_model_layer(const qfb_exec_plan* plan, int64_t n_act, int64_t c_out,
                                int64_t per, int32_t weights_cached, int32_t fused_fails,
                                qfb_exec_trace* delta);

/* ---------------------------------------------------------------------- */
/* Frame-level host pass: the quant portion of run_frontend +             */
/* backward_train (exec.hpp:435-451, frontend.hpp:236-258) for a set of    */
/* quant points given as HOST float32 buffers. Each input tensor is copied */
/* once even when it feeds two consumers; host->device copies, kernels and */
/* device->host copies are pipelined over two copy engines and the       */
/* compute stream, in groups of points (~80 MB of input each). Pinned host */
/* buffers get full PCIe bandwidth; pageable ones work too (driver-staged).*/
/* Copies that are contiguous on both sides are merged into one DMA        */
/* operation, so a caller whose buffers are carved from two pinned arenas  */
/* in copy order — inputs: per point x, then each consumer's up; outputs:  */
/* per point and consumer y, then dx (16-byte aligned offsets) — moves a   */
/* frame in a handful of copies. Synchronous. Results are identical to the */
/* per-point *_host calls.                                                  */
/* ---------------------------------------------------------------------- */
typedef struct qfb_host_point {
  const float* x;                              /* [outer, channels, inner] */
  int64_t outer, channels, inner;
  int32_t n_out;                               /* consumers: 1 or 2        */
  int32_t reserved;
  const double* s[QFB_MAX_CHAIN_OUT];          /* fwd scales [channels]    */
  float* y[QFB_MAX_CHAIN_OUT];                 /* fwd outputs (nullable)   */
  const double* log_s[QFB_MAX_CHAIN_OUT];      /* bwd log scales (nullable: no bwd) */
  const float* up[QFB_MAX_CHAIN_OUT];          /* bwd upstream             */
  float* dx[QFB_MAX_CHAIN_OUT];                /* d_input (nullable)       */
  double* d_log_s[QFB_MAX_CHAIN_OUT];          /* scale gradients [channels] */
} qfb_host_point;

qfb_status qfb_quant_pass_host(qfb_ctx* ctx, qfb_precision prec,
                               const qfb_host_point* points, int32_t n,
                               const qfb_quant_config* cfg);
/* The same pass split in two so consecutive frames overlap (frame k+1's   */
/* uploads run under frame k's downloads): submit enqueues everything on  */
/* in-flight slot 0 or 1 and returns; wait blocks until that slot's       */
/* outputs are in the host buffers, copies its scale gradients out and    */
/* reports errors. Host buffers of a slot must stay valid and untouched   */
/* until its wait. qfb_quant_pass_host == submit(slot 0) + wait(slot 0).  */
qfb_status qfb_quant_pass_host_submit(qfb_ctx* ctx, qfb_precision prec,
                                      const qfb_host_point* points, int32_t n,
                                      const qfb_quant_config* cfg, int32_t slot);
qfb_status qfb_quant_pass_host_wait(qfb_ctx* ctx, int32_t slot);


/* ---------------------------------------------------------------------- */
/* Scale-only QAT step pieces on the device — SURVEY.md §8 f3.            */
/* ---------------------------------------------------------------------- */
/* One tensor pair of qf::distill_loss (pair_loss, distill.hpp:66-124):     */
/* student/teacher are DEVICE float32 [channels, hw]; writes d_student      */
/* (= the reference's d_s, then scaled float(d * grad_scale) like the      */
/* trainer's 1/chunk_len scaling, distill.hpp:243-246; 1.0 = none) and     */
/* out2 (DEVICE double[2]) = {mse, mean per-location cosine}. Bit-exact:    */
/* the MSE and the cosine mean use the reference's pairwise tree.          */
qfb_status qfb_distill_pair(qfb_ctx* ctx, const float* student, const float* teacher,
                            int64_t channels, int64_t hw, double lambda_cos,
                            double grad_scale, float* d_student, double* out2);
/* The same for `pairs` independent pairs of one shape stored back to back */
/* ([pairs, channels, hw], e.g. the frames of a chunk), in one set of     */
/* launches; out (DEVICE double[pairs][2]).                               */
qfb_status qfb_distill_batch(qfb_ctx* ctx, const float* student, const float* teacher,
                             int64_t pairs, int64_t channels, int64_t hw, double lambda_cos,
                             double grad_scale, float* d_student, double* out);
/* qf::distill_loss (distill.hpp:126-141) on HOST buffers: out5 = {total,   */
/* mse_f, mse_i, cos_f, cos_i}; d_features / d_descriptors host float32.   */
qfb_status qfb_distill_loss_host(qfb_ctx* ctx, const float* f_s, const float* f_t,
                                 int64_t f_channels, int64_t f_hw, const float* i_s,
                                 const float* i_t, int64_t i_channels, int64_t i_hw,
                                 double lambda_cos, double grad_scale, double* out5,
                                 float* d_features, float* d_descriptors);
/* Adam over the flattened scale vector (distill.hpp:264-279), all DEVICE  */
/* double arrays. bc1/bc2 = 1 - beta^t from qfb_adam_bias_corrections (the */
/* host libm pow, like the reference). A non-finite gradient skips the     */
/* whole update (grads.all_finite(), distill.hpp:254-258): *skipped        */
/* (DEVICE u32) = number of non-finite gradients, 0 when applied.          */
/* Row-order fold of nrows gradient rows [nrows, n] (DEVICE doubles):     */
/* out = ((into + r0) + r1) + ... (into nullable: r0 + r1 + ...) — the    */
/* combine step of the multi-GPU scale-gradient exchange, bit-identical   */
/* to the trainer's frame-order accumulation (frontend.hpp:222-228).      */
qfb_status qfb_fold_rows(qfb_ctx* ctx, const double* rows, int64_t nrows, int64_t n,
                         const double* into, double* out);
/* ---- multi-GPU scale-gradient exchange ----------------- */
/* NCCL is loaded at run time (dlopen: the copy already in the process,    */
/* else libnccl.so.2 / $QFB_NCCL_LIB); without it these return            */
/* QFB_ERR_NCCL. `comm` is an ncclComm_t (void* here: no NCCL types in    */
/* the ABI). The step's one exchange replaces the trainer's in-process    */
/* `g += grad` over a chunk's frames (distill.hpp:249-250,                */
/* frontend.hpp:222-228) when the frames are sharded over GPUs.           */
qfb_status qfb_nccl_available(void);
/* ncclCommInitAll: one communicator per device, single process, one      */
/* stream per GPU (the process model of SURVEY §8e; no launcher needed).  */
qfb_status qfb_nccl_comm_init_all(int ndev, const int* devices, void** comms);
/* One process per GPU (torchrun / mpirun style): rank 0 creates the id,  */
/* the launcher's plumbing broadcasts its QFB_NCCL_UNIQUE_ID_BYTES bytes, */
/* every rank calls ncclCommInitRank on its device.                       */
#define QFB_NCCL_UNIQUE_ID_BYTES 128
qfb_status qfb_nccl_get_unique_id(void* id);
qfb_status qfb_nccl_comm_init_rank(void** comm, int nranks, const void* id, int rank,
                                   int device);
qfb_status qfb_nccl_comm_destroy(void* comm);
/* In-place ncclAllReduce(sum) of n DEVICE doubles on the context stream  */
/* (the cheap exchange; its bits depend on the GPU count).                */
qfb_status qfb_allreduce_scale_grads(qfb_ctx* ctx, void* comm, double* grads, int64_t n);
/* Bit-stable exchange: ncclAllGather of each rank's rows [rows_per_rank, */
/* n] into gathered [nranks * rows_per_rank, n] (rank-major = frame order */
/* when rank k holds frames k*rows_per_rank ...), then qfb_fold_rows      */
/* (into nullable): identical bits at every GPU count.                     */
qfb_status qfb_gather_fold_scale_grads(qfb_ctx* ctx, void* comm, const double* rows,
                                       int64_t rows_per_rank, int64_t n, double* gathered,
                                       const double* into, double* out);
qfb_status qfb_adam_bias_corrections(double beta1, double beta2, int64_t t,
                                     double* bc1, double* bc2);
qfb_status qfb_adam_step(qfb_ctx* ctx, double* params, double* m, double* v,
                         const double* grads, int64_t n, double beta1, double beta2,
                         double lr, double eps, double bc1, double bc2, uint32_t* skipped);
/* Graph-replayable Adam: the step counter lives on the DEVICE.           */
/* counters (DEVICE int64[3]) = {non-skipped steps, skipped steps,        */
/* table overflow}; t = counters[0] + 1 (distill.hpp:262-264); bc1/bc2 =  */
/* bias_table[2(t-1)], [2(t-1)+1] (DEVICE, from qfb_adam_bias_table: the  */
/* host libm pow, like the reference). The update is skipped (counters[1] */
/* += 1) when a gradient or one of the n_loss loss values is non-finite   */
/* (distill.hpp:254-258) or t > t_max; flag (DEVICE u32) = the count.     */
qfb_status qfb_adam_bias_table(double beta1, double beta2, int64_t t_max, double* table);
qfb_status qfb_adam_step_dev(qfb_ctx* ctx, double* params, double* m, double* v,
                             const double* grads, int64_t n, double beta1, double beta2,
                             double lr, double eps, const double* bias_table, int64_t t_max,
                             int64_t* counters, const double* loss, int64_t n_loss,
                             uint32_t* flag);

/* ---------------------------------------------------------------------- */
/* On-disk formats (host only, no GPU needed) — SURVEY.md §8 f4.           */
/* QSIM tensors: tensor_io.hpp:1-125 (magic "QSIM", u32 version 1, u32     */
/* rank, u64 dims, u8 precision tag, little-endian float32). Several       */
/* tensors may be concatenated in one blob; qfb_qsim_parse advances        */
/* *offset past one tensor like qf::parse_tensor (tensor_io.hpp:68-99).   */
/* Errors are QFB_ERR_IO with the reference's IoError messages.            */
/* ---------------------------------------------------------------------- */
typedef struct qfb_tensor_file qfb_tensor_file;
qfb_status qfb_qsim_parse(const void* buf, size_t size, size_t* offset,
                          qfb_tensor_file** out);          /* parse_tensor :68  */
qfb_status qfb_qsim_load(const char* path, qfb_tensor_file** out);  /* load_tensor :119 */
qfb_status qfb_qsim_info(const qfb_tensor_file* t, int32_t* rank, const int64_t** shape,
                         int32_t* precision, int64_t* numel, const float** data);
void qfb_qsim_free(qfb_tensor_file* t);
/* Byte-identical to serialize_tensor (tensor_io.hpp:55-66); out == NULL  */
/* queries the size.                                                      */
qfb_status qfb_qsim_serialize(const float* data, int32_t rank, const int64_t* shape,
                              int32_t precision, char* out, size_t cap, size_t* size);
qfb_status qfb_qsim_save(const char* path, const float* data, int32_t rank,
                         const int64_t* shape, int32_t precision);  /* save_tensor :115 */

/* QSCL scale checkpoints: distill.hpp:287-362 (magic "QSCL", u32 version */
/* 1, u64 manifest length, JSON manifest, float32 log-scale payload).     */
/* Layers are exposed in name order (qf::ScaleSet is a std::map).         */
typedef struct qfb_scales qfb_scales;
qfb_status qfb_qscl_parse(const void* buf, size_t size, qfb_scales** out); /* parse_scales :324 */
qfb_status qfb_qscl_load(const char* path, qfb_scales** out);               /* load_scales :360 */
int32_t qfb_qscl_count(const qfb_scales* s);
qfb_status qfb_qscl_layer(const qfb_scales* s, int32_t i, const char** name,
                          const double** log_w, int64_t* count, double* log_a);
void qfb_qscl_free(qfb_scales* s);
/* Byte-identical to serialize_scales (distill.hpp:296-318): layers in   */
/* name order, log scales stored as float32.                              */
qfb_status qfb_qscl_serialize(int32_t n, const char* const* names,
                              const double* const* log_w, const int64_t* counts,
                              const double* log_a, char* out, size_t cap, size_t* size);
qfb_status qfb_qscl_save(const char* path, int32_t n, const char* const* names,
                         const double* const* log_w, const int64_t* counts,
                         const double* log_a);                      /* save_scales :320 */

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* QFB_H_ */
