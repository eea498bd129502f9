// qfb_api.cpp — the C-ABI (include/qfb.h): argument validation (before
// anything is enqueued, like the reference's throw-before-compute),
// host-side scale math with the host libm, the per-(device, stream)
// context with its self-resetting reduction workspace, and launch planning
// (vector/scalar path choice, descriptor tables, grid sizing).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/qfb.h"
#include "qfb_kernels.h"

using namespace qfb;

namespace {

thread_local std::string g_last_error;

qfb_status fail(qfb_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

}  // namespace

// Shared with the other host TUs (qfb_formats.cpp, qfb_train.cpp).
qfb_status qfb::set_error(qfb_status st, const char* msg) {
  g_last_error = msg;
  return st;
}

namespace {

qfb_status cuda_fail(cudaError_t e, const char* where) {
  return fail(QFB_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define QFB_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

// Scoped device switch so calls from any thread land on the ctx device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Device buffer that only grows.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct qfb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  int ew_blocks_per_sm[2][2] = {{4, 4}, {4, 4}};  // [dtype][chain]
  int bwd_blocks_per_sm[2] = {4, 4};
  int tma_blocks_per_sm[2][2][kTmaStagesMax + 1] = {};  // [dtype][chain][stages]; 0: unavailable
  int tma_stages_env = 0;  // QFB_FWD_STAGES: fixed ring depth (tuning sweeps)
  uint32_t fwd_chunk_units = 0;  // QFB_FWD_CHUNK: TMA chunk size in 16-byte units (0: kEwChunk)
  std::vector<std::pair<size_t, int>> bwd_occ[2];  // (smem, blocks/SM) cache
  uint32_t* d_status = nullptr;
  uint32_t* h_status = nullptr;  // pinned
  DevBuf ws_f64;                 // partials / segment results
  DevBuf ws_u32;                 // tickets (kept zero between launches)
  DevBuf host_io[6];             // scratch for the *_host entry points
  int64_t launches = 0;
  // qfb_quant_pass_host: copy streams and, per in-flight slot, events,
  // per-point device buffers and pinned staging
  cudaStream_t s_in = nullptr, s_out = nullptr;
  struct PassSlot {
    std::vector<cudaEvent_t> ev;
    // device buffers of the pass: one input arena (per point: x, then the
    // consumers' upstreams) and one output arena (per point and consumer:
    // y, then d_input), laid out in copy order, so a caller whose host
    // buffers are laid out the same way gets its copies merged
    DevBuf in_arena, out_arena;
    std::vector<void*> ptr;  // per point: x, up[2], y[2], dx[2] (7 slots)
    DevBuf params;
    void* pinned = nullptr;  // params up, scale gradients and the status word down
    size_t pinned_bytes = 0;
    cudaEvent_t done = nullptr;  // after the slot's last download
    bool busy = false;
    // what wait() hands back: d_log_s destinations and their offsets in pinned
    std::vector<std::pair<double*, size_t>> grads;
    std::vector<int64_t> grad_len;
    uint32_t* h_status = nullptr;  // inside pinned
    const double* grad_base = nullptr;  // the pinned double block
  } slots[2];
  DevBuf train_ws[4];      // scratch of the trainer ops (qfb_train.cu)
  // buffers replaced by grow(): a captured graph may still reference them
  std::vector<void*> retired;
  // streaming backward: per row length, the device table of per-chunk block
  // metadata (kSbMetaWords u32 per chunk of a row); never freed before
  // qfb_ctx_destroy (captured graphs hold the pointers)
  struct SbShape {
    uint32_t* meta = nullptr;
    uint32_t nch = 0;
  };
  std::vector<std::pair<uint64_t, SbShape>> sb_shapes;
  int sb_blocks_per_sm[2] = {0, 0};
  // backward kernel (QFB_BWD_IMPL at creation): 0 tile kernel with
  // consumer-side partials (default), 1 tile kernel as in round 1 ("tile1"),
  // 2 streaming kernel ("stream")
  int bwd_impl = 0;
  // consumer layout of the full-tile kernel (QFB_BWD_IMPL=tile[q][m][d] at creation)
  uint32_t bwd_layout = kBwdLayoutDD;  // measured best (r02)
  // tile order of the full-tile kernel (QFB_BWD_ORDER=rev|fwd at creation):
  // last tile first by default — in a forward/backward step the backward
  // then starts on the points whose inputs the forward read last (partly
  // still in L2): f32 step 0.1326 -> 0.1311 ms (r02bg)
  uint32_t bwd_order = kBwdLayoutReverse;
  bool bwd_half_fp32 = false;           // QFB_OPT_BWD_HALF_FP32
  cudaEvent_t main_pass_event = nullptr;  // QFB_OPT_MAIN_PASS_EVENT
  // QFB_OPT_BWD_ASYNC_FINISH: side stream for the finisher, fork/join events
  bool async_finish = false;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool side_pending = false;
  // status word the forward kernels latch into: d_status, or a host-pass
  // slot's own word while that slot's kernels are enqueued
  uint32_t* cur_status = nullptr;
};

namespace {

// Grow a workspace buffer. The old buffer is NOT freed: a CUDA graph
// captured earlier may hold its address (baked into a __grid_constant__
// descriptor), so it is retired and freed only by qfb_ctx_destroy (growth
// is geometric, so the retired total stays below the live size). Growth
// during a stream capture is refused: cudaMalloc is not capturable, and the
// caller must size the context first (an eager call, or *_reserve).
qfb_status grow(qfb_ctx* ctx, DevBuf& b, size_t bytes, bool zero) {
  if (b.bytes >= bytes) return QFB_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(ctx->stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
    return fail(QFB_ERR_UNSUPPORTED,
                "workspace must grow to %zu bytes during a stream capture: run the call once eagerly "
                "(or qfb_fq_bwd_reserve) before capturing", bytes);
  size_t nb = std::max(bytes, b.bytes * 2);
  nb = (nb + 255) & ~size_t(255);
  void* np = nullptr;
  QFB_CUDA(cudaMalloc(&np, nb));
  if (zero) QFB_CUDA(cudaMemsetAsync(np, 0, nb, ctx->stream));
  if (b.p) ctx->retired.push_back(b.p);
  b.p = np;
  b.bytes = nb;
  return QFB_OK;
}

}  // namespace

// ---- internal accessors for the other TUs (qfb_kernels.h) ----
qfb_status qfb::ctx_scratch(qfb_ctx* ctx, int slot, size_t bytes, void** p) {
  if (!ctx) return fail(QFB_ERR_VALUE, "null qfb_ctx");
  if (slot < 0 || slot >= 4) return fail(QFB_ERR_VALUE, "scratch slot out of range");
  if (qfb_status st = grow(ctx, ctx->train_ws[slot], std::max<size_t>(bytes, 8), false)) return st;
  *p = ctx->train_ws[slot].p;
  return QFB_OK;
}
cudaStream_t qfb::ctx_stream(const qfb_ctx* ctx) { return ctx->stream; }
int qfb::ctx_device(const qfb_ctx* ctx) { return ctx->device; }

bool qfb::pdl_enabled(int which) {
  static const int mask = [] {
    const char* e = getenv("QFB_PDL");
    return e ? atoi(e) : kPdlFin;
  }();
  return (mask & which) != 0;
}

cudaError_t qfb::launch_main(const void* fn, dim3 grid, dim3 block, void** args, size_t smem,
                             cudaStream_t st, int which) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled(which) ? 1 : 0;
  return cudaLaunchKernelExC(&cfg, fn, args);
}
void qfb::ctx_count_launches(qfb_ctx* ctx, int n) { ctx->launches += n; }
qfb_status qfb::cuda_error(cudaError_t e, const char* where) { return cuda_fail(e, where); }

namespace {

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

qfb_status check_ctx(qfb_ctx* ctx) {
  if (!ctx) return fail(QFB_ERR_VALUE, "null qfb_ctx");
  return QFB_OK;
}

// tensor.hpp:58-64: every dim must be positive.
qfb_status check_dims(int64_t outer, int64_t channels, int64_t inner, const char* who) {
  if (outer <= 0 || channels <= 0 || inner <= 0) {
    return fail(QFB_ERR_SHAPE, "%s: non-positive dim in shape [%lld,%lld,%lld]", who,
                (long long)outer, (long long)channels, (long long)inner);
  }
  if (outer > INT64_MAX / channels || outer * channels > INT64_MAX / inner) {
    return fail(QFB_ERR_SHAPE, "%s: element count overflows", who);
  }
  return QFB_OK;
}

qfb_status check_dtype(int dtype) {
  if (dtype != QFB_F32 && dtype != QFB_F16) return fail(QFB_ERR_VALUE, "unknown dtype %d", dtype);
  return QFB_OK;
}

int elem_size(int dtype) { return dtype == QFB_F32 ? 4 : 2; }
int per_vec(int dtype) { return dtype == QFB_F32 ? 4 : 8; }

// Streaming-backward ring depth (QFB_SB_STAGES = 2..4 overrides).
int sb_stages(int dtype) {
  static const int env = [] {
    const char* e = getenv("QFB_SB_STAGES");
    const int v = e ? atoi(e) : 0;
    return v >= 2 && v <= 4 ? v : 0;
  }();
  (void)dtype;
  return env ? env : 4;
}

constexpr uint64_t kMaxUnits = 1ull << 31;

// One logical elementwise job, before splitting into <2^31-unit pieces.
struct EwJob {
  const void* a;
  const void* b;
  void* preact;
  void* y[2];
  const float* s[2];
  int64_t outer, channels, inner;
  int n_out, act;
  uint32_t flags;
  float q;
};

// Split a job into descriptors: vector path when every pointer is 16-byte
// aligned and a vector never straddles a channel boundary.
qfb_status plan_ew(int dtype, const EwJob& j, std::vector<EwDesc>& out) {
  const int V = per_vec(dtype);
  const int es = elem_size(dtype);
  const int64_t row = j.channels * j.inner;  // elements per outer index
  const int64_t n = j.outer * row;
  bool vec = (j.channels == 1 ? (n % V == 0) : (j.inner % V == 0));
  vec = vec && aligned16(j.a) && (!j.b || aligned16(j.b)) && (!j.preact || aligned16(j.preact));
  for (int k = 0; k < j.n_out; ++k) vec = vec && aligned16(j.y[k]);
  const int64_t unit = vec ? V : 1;
  // Rows per piece so a piece stays below 2^31 units.
  int64_t rows_per_piece = j.outer;
  if ((uint64_t)(n / unit) >= kMaxUnits) {
    rows_per_piece = (int64_t)(kMaxUnits * (uint64_t)unit / (uint64_t)row);
    if (rows_per_piece == 0) {
      if (j.channels != 1) return fail(QFB_ERR_UNSUPPORTED, "row of %lld elements too large", (long long)row);
    }
  }
  auto emit = [&](int64_t elem_off, int64_t elems, int64_t inner_units, int64_t chans) {
    EwDesc d{};
    const char* base = nullptr;
    (void)base;
    d.a = static_cast<const char*>(j.a) + elem_off * es;
    d.b = j.b ? static_cast<const char*>(j.b) + elem_off * es : nullptr;
    d.preact = j.preact ? static_cast<char*>(j.preact) + elem_off * es : nullptr;
    for (int k = 0; k < 2; ++k) {
      // int8-code outputs are 1 byte per element
      const int oes = (j.flags & kEwInt8Out) ? 1 : es;
      d.y[k] = k < j.n_out ? static_cast<char*>(j.y[k]) + elem_off * oes : nullptr;
      d.s[k] = k < j.n_out ? j.s[k] : nullptr;
    }
    d.nunits = (uint32_t)(elems / unit);
    d.vec = (uint32_t)unit;
    d.inner_u = make_fastdiv((uint32_t)std::max<int64_t>(inner_units, 1));
    d.chans = make_fastdiv((uint32_t)chans);
    d.n_out = j.n_out;
    d.act = j.act;
    d.flags = j.flags;
    d.q = j.q;
    out.push_back(d);
  };
  if (j.channels == 1) {
    // per-tensor: split anywhere on a unit boundary
    const int64_t max_elems = (int64_t)(kMaxUnits / 2) * unit;
    for (int64_t off = 0; off < n; off += max_elems) {
      emit(off, std::min(max_elems, n - off), 1, 1);
    }
    return QFB_OK;
  }
  if (j.inner / unit >= (int64_t)UINT32_MAX || j.channels >= (int64_t)UINT32_MAX) {
    return fail(QFB_ERR_UNSUPPORTED, "inner/channels too large");
  }
  for (int64_t r = 0; r < j.outer; r += rows_per_piece) {
    const int64_t rows = std::min(rows_per_piece, j.outer - r);
    emit(r * row, rows * row, j.inner / unit, j.channels);
  }
  return QFB_OK;
}

// TMA ring depth for one launch (measured on B200). Bytes in
// flight per SM with 16 KB chunks: 2 stages x 5 CTAs -> 80 KB, 3 x 4 ->
// 128 KB, 4 x 3 -> 144 KB. Deeper rings fill and drain slower and leave a
// longer one-chunk tail, so short launches (one frame) take 3 stages and
// long ones (>= 64 chunks per CTA, e.g. 8 frames) 4. Chains stage two
// arrays per chunk and keep 2 stages; f16 and int8-code emission are
// element-rate bound and want the most CTAs (2 stages).
int tma_stages(const qfb_ctx* ctx, int dtype, bool chain, bool int8_out, uint64_t chunks) {
  if (ctx->tma_stages_env) return ctx->tma_stages_env;
  if (chain || int8_out) return 2;
  if (dtype != 0) {
    // f16 plain: 3 stages for medium launches (one frame: 36.3 -> 35.8 us),
    // 2 for long ones (8 frames: 0.222 vs 0.226 ms) and tiny ones
    const uint64_t ctas2h = (uint64_t)ctx->sm_count * (uint64_t)std::max(1, ctx->tma_blocks_per_sm[dtype][0][2]);
    return (chunks >= 2 * ctas2h && chunks < 32 * ctas2h) ? 3 : 2;
  }
  // short launches (about one chunk per CTA, e.g. one 128x120x160 map): the
  // 2-stage ring's extra CTAs beat depth (6.5 -> 6.0 us per call; with PDL
  // on these launches the early-scheduled dependents take those CTA slots
  // and it is 6.6, so kPdlFwdSmall stays off by default)
  const uint64_t ctas2 = (uint64_t)ctx->sm_count * (uint64_t)std::max(1, ctx->tma_blocks_per_sm[dtype][0][2]);
  if (chunks < 2 * ctas2) return 2;
  const uint64_t ctas4 = (uint64_t)ctx->sm_count * (uint64_t)std::max(1, ctx->tma_blocks_per_sm[dtype][0][4]);
  return chunks >= 64 * ctas4 ? 4 : 3;
}

qfb_status run_ew(qfb_ctx* ctx, int dtype, const std::vector<EwDesc>& descs, bool chain) {
  size_t i = 0;
  while (i < descs.size()) {
    EwBatch b;
    std::memset(&b, 0, sizeof b);
    uint32_t chunks = 0;
    int n = 0;
    for (; i < descs.size() && n < kMaxEwDesc; ++i, ++n) {
      b.d[n] = descs[i];
      b.chunk_begin[n] = chunks;
      chunks += (descs[i].nunits + kEwChunk - 1) / kEwChunk;
    }
    b.n = n;
    b.chunk_begin[n] = chunks;
    b.chunk_units = (uint32_t)kEwChunk;
    if (chunks == 0) continue;
    bool int8_out = false;
    for (int k = 0; k < n; ++k) int8_out = int8_out || (b.d[k].flags & kEwInt8Out) != 0;
    const int stages = tma_stages(ctx, dtype, chain, int8_out, chunks);
    const int tma_per_sm = ctx->tma_blocks_per_sm[dtype][chain ? 1 : 0][stages];
    bool all_vec = tma_per_sm > 0;
    for (int k = 0; k < n && all_vec; ++k) all_vec = b.d[k].vec > 1;
    cudaError_t e;
    if (all_vec && ctx->fwd_chunk_units > 0 && ctx->fwd_chunk_units < (uint32_t)kEwChunk) {
      // smaller TMA chunks (QFB_FWD_CHUNK): the table in those units
      const uint32_t cu = ctx->fwd_chunk_units;
      b.chunk_units = cu;
      chunks = 0;
      for (int k = 0; k < n; ++k) {
        b.chunk_begin[k] = chunks;
        chunks += (b.d[k].nunits + cu - 1) / cu;
      }
      b.chunk_begin[n] = chunks;
    }
    if (all_vec) {
      const int grid = (int)std::min<uint64_t>(chunks, (uint64_t)ctx->sm_count * tma_per_sm);
      e = launch_ew_tma(dtype, chain, stages, b, ctx->cur_status, grid, ctx->stream,
                        chunks < 4ull * (uint64_t)grid);
    } else {
      const int grid = (int)std::min<uint64_t>(
          chunks, (uint64_t)ctx->sm_count * ctx->ew_blocks_per_sm[dtype][chain ? 1 : 0]);
      e = launch_ew(dtype, chain, b, ctx->cur_status, grid, ctx->stream);
    }
    if (e != cudaSuccess) return cuda_fail(e, "ew_kernel launch");
    ctx->launches++;
  }
  return QFB_OK;
}

qfb_status q_of(int32_t q_max, float* q) {
  if (q_max < 1 || q_max > 32767) return fail(QFB_ERR_VALUE, "q_max %d out of range", q_max);
  *q = (float)q_max;
  return QFB_OK;
}

}  // namespace

// =====================================================================
extern "C" {

const char* qfb_last_error(void) { return g_last_error.c_str(); }

const char* qfb_status_name(qfb_status s) {
  switch (s) {
    case QFB_OK: return "OK";
    case QFB_ERR_SHAPE: return "ShapeError";
    case QFB_ERR_VALUE: return "ValueError";
    case QFB_ERR_IO: return "IoError";
    case QFB_ERR_NONFINITE: return "NonFiniteError";
    case QFB_ERR_INSUFFICIENT: return "InsufficientMatchesError";
    case QFB_ERR_FUSED_PATH: return "FusedPathError";
    case QFB_ERR_CUDA: return "CudaError";
    case QFB_ERR_NCCL: return "NcclError";
    case QFB_ERR_UNSUPPORTED: return "Unsupported";
  }
  return "Unknown";
}

const char* qfb_build_info(void) {
  return "qfb 0.1 sm_100a (compute_100a) ieee-div ftz=off no-fast-math";
}

// ----------------------------------------------------------- config ---
void qfb_quant_config_default(qfb_quant_config* c) {
  if (!c) return;
  c->bits = 8;
  c->reserved = 0;
  c->s_min = 1e-6;
  c->s_min_half = 1e-4;
  c->s_max = 64.0;
  c->eps = 1e-8;
}

qfb_status qfb_quant_config_validate(const qfb_quant_config* c) {
  if (!c) return fail(QFB_ERR_VALUE, "null config");
  if (c->bits < 2 || c->bits > 16) return fail(QFB_ERR_VALUE, "QuantConfig: bits out of range");
  if (!(c->s_min > 0.0) || !(c->s_min < c->s_max))
    return fail(QFB_ERR_VALUE, "QuantConfig: require 0 < s_min < s_max");
  if (!(c->eps > 0.0) || !(c->eps < c->s_min))
    return fail(QFB_ERR_VALUE, "QuantConfig: require 0 < eps < s_min");
  if (!(c->s_min_half > 0.0) || !(c->s_min_half < c->s_max))
    return fail(QFB_ERR_VALUE, "QuantConfig: require 0 < s_min_half < s_max");
  return QFB_OK;
}

int32_t qfb_q_max(const qfb_quant_config* c) { return c ? (1 << (c->bits - 1)) - 1 : 127; }

// ------------------------------------------------------- scale math ---
// Same expressions as quant.hpp:71-109 evaluated with the host libm, so the
// doubles are bit-identical to the reference's on the same machine.
double qfb_softplus(double x) {
  if (x > 30.0) return x + std::log1p(std::exp(-x));
  return std::log1p(std::exp(x));
}

double qfb_sigmoid(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
  const double e = std::exp(x);
  return e / (1.0 + e);
}

qfb_status qfb_softplus_inv(double y, double* out) {
  if (!out) return fail(QFB_ERR_VALUE, "null output");
  if (!(y > 0.0)) return fail(QFB_ERR_VALUE, "softplus_inv: argument must be positive");
  *out = y > 30.0 ? y : std::log(std::expm1(y));
  return QFB_OK;
}

static double lower_for(const qfb_quant_config* c, qfb_precision p) {
  return p == QFB_PREC_HALF ? c->s_min_half : c->s_min;
}

qfb_status qfb_resolve_scales(const double* log_s, int64_t n, const qfb_quant_config* cfg,
                              qfb_precision prec, double* s_out) {
  if (n < 0 || (n > 0 && (!log_s || !s_out)) || !cfg) return fail(QFB_ERR_VALUE, "resolve_scales: bad args");
  const double lo = lower_for(cfg, prec);
  for (int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(log_s[i]))
      return fail(QFB_ERR_NONFINITE, "resolve_scale: non-finite log scale at %lld", (long long)i);
    const double raw = qfb_softplus(log_s[i]) + cfg->eps;
    s_out[i] = std::min(std::max(raw, lo), cfg->s_max);
  }
  return QFB_OK;
}

qfb_status qfb_scale_grad_factors(const double* log_s, int64_t n, const qfb_quant_config* cfg,
                                  qfb_precision prec, double* s_out, double* chain_out) {
  qfb_status st = qfb_resolve_scales(log_s, n, cfg, prec, s_out);
  if (st != QFB_OK) return st;
  if (!chain_out) return fail(QFB_ERR_VALUE, "scale_grad_factors: null chain");
  const double lo = lower_for(cfg, prec);
  for (int64_t i = 0; i < n; ++i) {
    const double raw = qfb_softplus(log_s[i]) + cfg->eps;  // quant.hpp:242-244
    const bool clamped = !(raw > lo && raw < cfg->s_max);
    chain_out[i] = clamped ? 0.0 : qfb_sigmoid(log_s[i]);
  }
  return QFB_OK;
}

qfb_status qfb_cast_scales_f32(const double* s, int64_t n, float* out) {
  if (n < 0 || (n > 0 && (!s || !out))) return fail(QFB_ERR_VALUE, "cast_scales: bad args");
  for (int64_t i = 0; i < n; ++i) {
    if (!(s[i] > 0.0))
      return fail(QFB_ERR_VALUE, "fake_quantize: scale must be positive, got %f", s[i]);
    out[i] = static_cast<float>(s[i]);
  }
  return QFB_OK;
}

// ---------------------------------------------------------- context ---
qfb_status qfb_ctx_create(int32_t device, void* stream, qfb_ctx** out) {
  if (!out) return fail(QFB_ERR_VALUE, "null out");
  *out = nullptr;
  int ndev = 0;
  QFB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(QFB_ERR_VALUE, "device %d out of range (%d)", device, ndev);
  DeviceGuard g(device);
  qfb_ctx* c = new qfb_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) {
    // occupancy of each elementwise kernel variant sizes its persistent grid
    for (int dt = 0; dt < 2; ++dt)
      for (int ch = 0; ch < 2; ++ch) {
        int per = 0;
        if (ew_occupancy(dt, ch != 0, &per) == cudaSuccess && per > 0) c->ew_blocks_per_sm[dt][ch] = per;
      }
    for (int dt = 0; dt < 2; ++dt) {
      int per = 0;
      if (bwd_occupancy(dt, &per) == cudaSuccess && per > 0) c->bwd_blocks_per_sm[dt] = per;
      for (int ch = 0; ch < 2; ++ch)
        for (int ns = kTmaStagesMin; ns <= kTmaStagesMax; ++ns) {
          per = 0;
          if (ew_tma_occupancy(dt, ch != 0, ns, &per) == cudaSuccess && per > 0)
            c->tma_blocks_per_sm[dt][ch][ns] = per;
        }
    }
    for (int dt = 0; dt < 2; ++dt) {
      int per = 0;
      if (sbwd_occupancy(dt, sb_stages(dt), &per) == cudaSuccess && per > 0) c->sb_blocks_per_sm[dt] = per;
    }
    if (const char* env = getenv("QFB_BWD_IMPL")) {
      c->bwd_impl = std::strcmp(env, "stream") == 0 ? 2 : std::strcmp(env, "tile1") == 0 ? 1 : 0;
      // consumer layout of the full-tile kernel (A/B runs and per-layout
      // tests): "tile" + any of q (quad), m (magic rint), d (dd quotient)
      if (std::strncmp(env, "tile", 4) == 0 && env[4] != '1') {
        uint32_t l = 0;
        for (const char* p = env + 4; *p; ++p) {
          l |= *p == 'q' ? kBwdLayoutQuad : *p == 'm' ? kBwdLayoutMagic : *p == 'd' ? kBwdLayoutDD
             : *p == '2' ? kBwdLayoutTwoCtas : *p == 'p' ? kBwdLayoutPrefetch : *p == 'u' ? kBwdLayoutCU : 0u;
        }
        c->bwd_layout = l;
      }
    }
    if (const char* env = getenv("QFB_BWD_ORDER")) c->bwd_order = std::strcmp(env, "fwd") == 0 ? 0u : kBwdLayoutReverse;
    if (const char* env = getenv("QFB_DISABLE_TMA_FWD"))
      if (env[0] == '1') std::memset(c->tma_blocks_per_sm, 0, sizeof c->tma_blocks_per_sm);
    if (const char* env = getenv("QFB_FWD_CHUNK")) {
      const int v = atoi(env);
      if (v >= 256 && v <= kEwChunk) c->fwd_chunk_units = (uint32_t)v;
    }
    if (const char* env = getenv("QFB_FWD_STAGES")) {
      const int v = atoi(env);
      if (v >= kTmaStagesMin && v <= kTmaStagesMax) c->tma_stages_env = v;
    }
  }
  // status words: [0] the context's, [1 + k] host-pass slot k's own
  if (e == cudaSuccess) e = cudaMalloc(&c->d_status, 3 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_status, sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemsetAsync(c->d_status, 0, 3 * sizeof(uint32_t), c->stream);
  c->cur_status = c->d_status;
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    qfb_ctx_destroy(c);
    return cuda_fail(e, "qfb_ctx_create");
  }
  *out = c;
  return QFB_OK;
}

qfb_status qfb_ctx_destroy(qfb_ctx* ctx) {
  if (!ctx) return QFB_OK;
  DeviceGuard g(ctx->device);
  // the host pass's copy streams may still move a slot's buffers
  cudaStreamSynchronize(ctx->stream);
  if (ctx->s_in) cudaStreamSynchronize(ctx->s_in);
  if (ctx->s_out) cudaStreamSynchronize(ctx->s_out);
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->ws_f64.p) cudaFree(ctx->ws_f64.p);
  if (ctx->ws_u32.p) cudaFree(ctx->ws_u32.p);
  for (void* p : ctx->retired) cudaFree(p);
  for (auto& kv : ctx->sb_shapes) cudaFree(kv.second.meta);
  for (auto& b : ctx->host_io)
    if (b.p) cudaFree(b.p);
  for (auto& b : ctx->train_ws)
    if (b.p) cudaFree(b.p);
  for (auto& sl : ctx->slots) {
    if (sl.in_arena.p) cudaFree(sl.in_arena.p);
    if (sl.out_arena.p) cudaFree(sl.out_arena.p);
    if (sl.params.p) cudaFree(sl.params.p);
    if (sl.pinned) cudaFreeHost(sl.pinned);
    for (auto e : sl.ev) cudaEventDestroy(e);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
  if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
  delete ctx;
  return QFB_OK;
}

qfb_status qfb_ctx_set_option(qfb_ctx* ctx, int32_t option, int64_t value) {
  if (qfb_status st = check_ctx(ctx)) return st;
  switch (option) {
    case QFB_OPT_BWD_HALF_FP32:
      if (value != 0 && value != 1) return fail(QFB_ERR_VALUE, "QFB_OPT_BWD_HALF_FP32 takes 0 or 1");
      ctx->bwd_half_fp32 = value != 0;
      return QFB_OK;
    case QFB_OPT_BWD_ASYNC_FINISH: {
      if (value != 0 && value != 1) return fail(QFB_ERR_VALUE, "QFB_OPT_BWD_ASYNC_FINISH takes 0 or 1");
      if (value && !ctx->side) {
        DeviceGuard g(ctx->device);
        QFB_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        QFB_CUDA(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        QFB_CUDA(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
      }
      if (!value)
        if (qfb_status st = qfb_ctx_join(ctx)) return st;
      ctx->async_finish = value != 0;
      return QFB_OK;
    }
    case QFB_OPT_MAIN_PASS_EVENT:
      ctx->main_pass_event = reinterpret_cast<cudaEvent_t>(static_cast<intptr_t>(value));
      return QFB_OK;
    default:
      return fail(QFB_ERR_VALUE, "unknown context option %d", option);
  }
}

qfb_status qfb_ctx_set_stream(qfb_ctx* ctx, void* stream) {
  if (qfb_status st = check_ctx(ctx)) return st;
  ctx->stream = static_cast<cudaStream_t>(stream);
  return QFB_OK;
}

void* qfb_ctx_stream(qfb_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
int32_t qfb_ctx_sm_count(qfb_ctx* ctx) { return ctx ? ctx->sm_count : 0; }
int64_t qfb_ctx_launch_count(qfb_ctx* ctx) { return ctx ? ctx->launches : 0; }

qfb_status qfb_ctx_join(qfb_ctx* ctx) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (!ctx->side_pending) return QFB_OK;
  DeviceGuard g(ctx->device);
  QFB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
  ctx->side_pending = false;
  return QFB_OK;
}

qfb_status qfb_ctx_sync(qfb_ctx* ctx) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = qfb_ctx_join(ctx)) return st;
  DeviceGuard g(ctx->device);
  QFB_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           ctx->stream));
  QFB_CUDA(cudaStreamSynchronize(ctx->stream));
  const uint32_t flags = *ctx->h_status;
  if (flags != 0) {
    QFB_CUDA(cudaMemsetAsync(ctx->d_status, 0, sizeof(uint32_t), ctx->stream));
    QFB_CUDA(cudaStreamSynchronize(ctx->stream));
    return fail(QFB_ERR_NONFINITE, "demote_half: non-finite value on the binary16 path");
  }
  return QFB_OK;
}

// --------------------------------------------------- forward ops ---
qfb_status qfb_fq_fwd(qfb_ctx* ctx, qfb_dtype dtype, const void* x, void* y, int64_t outer,
                      int64_t channels, int64_t inner, const float* scale, int32_t q_max,
                      uint32_t flags) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = check_dtype(dtype)) return st;
  if (qfb_status st = check_dims(outer, channels, inner, "fake_quantize")) return st;
  if (!x || !y || !scale) return fail(QFB_ERR_VALUE, "fake_quantize: null pointer");
  float q;
  if (qfb_status st = q_of(q_max, &q)) return st;
  EwJob j{x, nullptr, nullptr, {y, nullptr}, {scale, nullptr}, outer, channels, inner,
          1, QFB_ACT_NONE, flags & (kEwHalfGrid | kEwStreaming), q};
  std::vector<EwDesc> d;
  if (qfb_status st = plan_ew(dtype, j, d)) return st;
  DeviceGuard g(ctx->device);
  return run_ew(ctx, dtype, d, false);
}

qfb_status qfb_fq_fwd_multi(qfb_ctx* ctx, qfb_dtype dtype, const qfb_fq_desc* table, int32_t n) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = check_dtype(dtype)) return st;
  if (n < 0 || (n > 0 && !table)) return fail(QFB_ERR_VALUE, "fq_fwd_multi: bad table");
  std::vector<EwDesc> d;
  for (int32_t i = 0; i < n; ++i) {
    const qfb_fq_desc& t = table[i];
    if (qfb_status st = check_dims(t.outer, t.channels, t.inner, "fq_fwd_multi")) return st;
    if (t.n_out < 1 || t.n_out > 2) return fail(QFB_ERR_VALUE, "fq_fwd_multi: n_out must be 1 or 2");
    if (!t.x || !t.y[0] || !t.scale[0] || (t.n_out == 2 && (!t.y[1] || !t.scale[1])))
      return fail(QFB_ERR_VALUE, "fq_fwd_multi: null pointer in entry %d", i);
    float q;
    if (qfb_status st = q_of(t.q_max, &q)) return st;
    EwJob j{t.x, nullptr, nullptr, {t.y[0], t.y[1]}, {t.scale[0], t.scale[1]}, t.outer,
            t.channels, t.inner, t.n_out, QFB_ACT_NONE,
            t.flags & (kEwHalfGrid | kEwStreaming | kEwInt8Out), q};
    if (qfb_status st = plan_ew(dtype, j, d)) return st;
  }
  DeviceGuard g(ctx->device);
  return run_ew(ctx, dtype, d, false);
}

static qfb_status chain_job(const qfb_chain_desc& t, EwJob& j) {
  if (qfb_status st = check_dtype(t.dtype)) return st;
  if (qfb_status st = check_dims(t.outer, t.channels, t.inner, "fq_chain")) return st;
  if (t.n_out < 0 || t.n_out > 2) return fail(QFB_ERR_VALUE, "fq_chain: n_out must be 0..2");
  if (t.act < 0 || t.act > 2) return fail(QFB_ERR_VALUE, "fq_chain: unknown activation %d", t.act);
  if (!t.a) return fail(QFB_ERR_VALUE, "fq_chain: null input");
  for (int k = 0; k < t.n_out; ++k)
    if (!t.y[k] || !t.scale[k]) return fail(QFB_ERR_VALUE, "fq_chain: null output %d", k);
  if (t.n_out == 0 && !t.preact) return fail(QFB_ERR_VALUE, "fq_chain: no outputs");
  float q;
  if (qfb_status st = q_of(t.q_max, &q)) return st;
  const bool half = t.dtype == QFB_F16 || (t.flags & QFB_FLAG_HALF_GRID);
  uint32_t flags = t.flags & (kEwHalfGrid | kEwStreaming);
  if (half) flags |= kEwDemoteIn;
  j = EwJob{t.a, t.b, t.preact, {t.y[0], t.y[1]}, {t.scale[0], t.scale[1]}, t.outer,
            t.channels, t.inner, t.n_out, t.act, flags, q};
  return QFB_OK;
}

qfb_status qfb_fq_chain(qfb_ctx* ctx, const qfb_chain_desc* desc) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (!desc) return fail(QFB_ERR_VALUE, "fq_chain: null desc");
  return qfb_fq_chain_multi(ctx, desc, 1);
}

qfb_status qfb_fq_chain_multi(qfb_ctx* ctx, const qfb_chain_desc* table, int32_t n) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (n < 0 || (n > 0 && !table)) return fail(QFB_ERR_VALUE, "fq_chain_multi: bad table");
  // one launch per dtype group (a batch shares the element type)
  for (int dt = 0; dt < 2; ++dt) {
    std::vector<EwDesc> d;
    for (int32_t i = 0; i < n; ++i) {
      EwJob j;
      if (qfb_status st = chain_job(table[i], j)) return st;
      if (table[i].dtype != dt) continue;
      if (qfb_status st = plan_ew(dt, j, d)) return st;
    }
    if (d.empty()) continue;
    DeviceGuard g(ctx->device);
    if (qfb_status st = run_ew(ctx, dt, d, true)) return st;
  }
  return QFB_OK;
}

qfb_status qfb_int8_codes(qfb_ctx* ctx, qfb_dtype dtype, const void* x, int8_t* codes,
                          int64_t outer, int64_t channels, int64_t inner, const float* scale,
                          int32_t q_max) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = check_dtype(dtype)) return st;
  if (qfb_status st = check_dims(outer, channels, inner, "int8_codes")) return st;
  if (!x || !codes || !scale) return fail(QFB_ERR_VALUE, "int8_codes: null pointer");
  float q;
  if (qfb_status st = q_of(q_max, &q)) return st;
  const int V = per_vec(dtype);
  const int64_t n = outer * channels * inner;
  if (n >= (int64_t)kMaxUnits) return fail(QFB_ERR_UNSUPPORTED, "int8_codes: tensor too large");
  const bool vec = (channels == 1 ? n % V == 0 : inner % V == 0) && aligned16(x) &&
                   ((reinterpret_cast<uintptr_t>(codes) & (V - 1)) == 0);
  const int64_t unit = vec ? V : 1;
  CodesDesc d{};
  d.x = x;
  d.codes = codes;
  d.s = scale;
  d.nunits = (uint32_t)(n / unit);
  d.vec = (uint32_t)unit;
  d.inner_u = make_fastdiv((uint32_t)(inner / unit > 0 ? inner / unit : 1));
  d.chans = make_fastdiv((uint32_t)channels);
  d.q = q;
  DeviceGuard g(ctx->device);
  const int grid = (int)std::min<int64_t>((d.nunits + kEwThreads - 1) / kEwThreads,
                                          (int64_t)ctx->sm_count * 8);
  cudaError_t e = launch_codes(dtype, d, std::max(grid, 1), ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "codes_kernel launch");
  ctx->launches++;
  return QFB_OK;
}

qfb_status qfb_fq_fwd_perop(qfb_ctx* ctx, qfb_dtype dtype, const void* x, void* y,
                            int64_t outer, int64_t channels, int64_t inner, const float* scale,
                            int32_t q_max, uint32_t flags, float* tmp) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = check_dtype(dtype)) return st;
  if (qfb_status st = check_dims(outer, channels, inner, "fake_quantize_perop")) return st;
  if (!x || !y || !scale || !tmp) return fail(QFB_ERR_VALUE, "fake_quantize_perop: null pointer");
  float q;
  if (qfb_status st = q_of(q_max, &q)) return st;
  const uint64_t n = (uint64_t)(outer * channels * inner);
  float* t1 = tmp;
  float* t2 = tmp + n;
  float* t3 = tmp + 2 * n;
  const void* ins[4] = {x, t1, t2, t3};
  void* outs[4] = {t1, t2, t3, y};
  DeviceGuard g(ctx->device);
  const int grid = (int)std::min<uint64_t>((n + kEwThreads - 1) / kEwThreads,
                                           (uint64_t)ctx->sm_count * 8);
  for (int op = 0; op < 4; ++op) {
    PerOpDesc d{ins[op], outs[op], scale, n, (uint64_t)inner, (uint64_t)channels, q,
                flags & kEwHalfGrid};
    cudaError_t e = launch_perop(dtype, op, d, ctx->cur_status, std::max(grid, 1), ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "perop_kernel launch");
    ctx->launches++;
  }
  return QFB_OK;
}

qfb_status qfb_fill_rng(qfb_ctx* ctx, qfb_dtype dtype, void* out, int64_t n, uint64_t seed,
                        uint64_t stream, uint64_t index_offset, int32_t kind, double lo,
                        double hi) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = check_dtype(dtype)) return st;
  if (n < 0 || (n > 0 && !out)) return fail(QFB_ERR_VALUE, "fill_rng: bad args");
  if (kind != 0 && kind != 1) return fail(QFB_ERR_VALUE, "fill_rng: kind must be 0 or 1");
  if (n == 0) return QFB_OK;
  DeviceGuard g(ctx->device);
  const int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sm_count * 16);
  cudaError_t e = launch_fill_rng(dtype, out, n, seed, stream, index_offset, kind, lo, hi, grid,
                                  ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "fill_rng launch");
  ctx->launches++;
  return QFB_OK;
}

qfb_status qfb_resolve_scales_dev(qfb_ctx* ctx, const double* log_s, int64_t n,
                                  const qfb_quant_config* cfg, qfb_precision prec, float* s32,
                                  double* s64, double* chain) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = qfb_quant_config_validate(cfg)) return st;
  if (n < 0 || (n > 0 && !log_s)) return fail(QFB_ERR_VALUE, "resolve_scales_dev: bad args");
  if (n == 0) return QFB_OK;
  ResolveDesc d{log_s, s32, s64, chain, n, lower_for(cfg, prec), cfg->s_max, cfg->eps};
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_resolve(d, ctx->cur_status, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "resolve launch");
  ctx->launches++;
  return QFB_OK;
}

// -------------------------------------------------- backward ops ---
namespace {

struct BwdPlan {
  BwdDesc d;
  uint64_t tiles;
  size_t f64_need;  // doubles
  size_t u32_need;  // counters
};

// Depth D of the 16-bounded leaf groups: smallest D with ceil(n/2^D) <= 16.
uint32_t leaf_depth(uint64_t n) {
  uint32_t d = 0;
  while (((n + (1ull << d) - 1) >> d) > (uint64_t)kLeafMax) ++d;
  return d;
}

qfb_status plan_bwd(const qfb_bwd_desc& t, BwdPlan& p, int dtype_of_plan) {
  if (qfb_status st = check_dims(t.outer, t.channels, t.inner, "fake_quantize_backward")) return st;
  if (!t.x || !t.up || !t.scale64 || !t.chain || !t.d_log_s)
    return fail(QFB_ERR_VALUE, "fake_quantize_backward: null pointer");
  if (t.q_max < 1 || t.q_max > 32767) return fail(QFB_ERR_VALUE, "q_max out of range");
  const uint64_t segs = (uint64_t)t.outer * (uint64_t)t.channels;
  if (segs >= (1ull << 32)) return fail(QFB_ERR_UNSUPPORTED, "too many rows");
  std::memset(&p, 0, sizeof p);
  BwdDesc& d = p.d;
  d.x = t.x;
  d.up = t.up;
  d.dx = t.dx;
  d.s64 = t.scale64;
  d.chain = t.chain;
  d.d_log_s = t.d_log_s;
  d.inner = (uint64_t)t.inner;
  d.outer = (uint32_t)t.outer;
  d.chans = (uint32_t)t.channels;
  d.depth = leaf_depth((uint64_t)t.inner);
  d.g = std::min<uint32_t>(d.depth, (uint32_t)kBwdGroupsLog);
  d.tps_log = d.depth - d.g;
  d.part_log = d.tps_log;
  if (t.accumulate < 0 || t.accumulate > QFB_BWD_ROWS)
    return fail(QFB_ERR_VALUE, "fake_quantize_backward: accumulate must be 0, 1 or QFB_BWD_ROWS");
  if (t.row_stride < 0) return fail(QFB_ERR_VALUE, "fake_quantize_backward: negative row_stride");
  d.accumulate = t.accumulate;
  d.row_stride = t.row_stride > 0 ? (uint64_t)t.row_stride : (uint64_t)t.channels;
  d.q = (double)t.q_max;
  d.vec = (aligned16(t.x) && aligned16(t.up) && (!t.dx || aligned16(t.dx))) ? 1u : 0u;
  d.total_bytes = (uint64_t)t.outer * (uint64_t)t.channels * (uint64_t)t.inner *
                  (uint64_t)elem_size(dtype_of_plan);
  const uint64_t tps = 1ull << d.tps_log;
  p.tiles = segs * tps;
  if (p.tiles >= (1ull << 31)) return fail(QFB_ERR_UNSUPPORTED, "too many tiles");
  p.f64_need = segs * tps;  // tile partials, reduced by the finisher
  p.u32_need = 0;
  return QFB_OK;
}

}  // namespace

namespace {

// ---- streaming backward planning (sbwd_kernel, qfb_bwd.cu) ----
// Eligible: 16-byte aligned x / up / dx, rows that are 16-byte multiples of
// at least one chunk and below 2^28 elements. QFB_BWD_IMPL=tile (read at
// context creation) forces the tile kernel.

bool sb_eligible(const BwdPlan& p, int dtype) {
  const uint64_t es = (uint64_t)elem_size(dtype);
  return p.d.vec && (p.d.inner * es) % 16 == 0 && p.d.inner >= (uint64_t)kSbChunk &&
         p.d.inner < (1ull << 28) && p.d.depth >= (uint32_t)kSbBlockLog;
}

// Block starts of a row of n elements at depth L of the reference's split
// (tensor.hpp:100-109: left child floor(m/2)); lo[2^L] = n.
std::vector<uint32_t> tree_starts(uint64_t n, uint32_t L) {
  std::vector<uint64_t> lo{0}, m{n};
  for (uint32_t l = 0; l < L; ++l) {
    std::vector<uint64_t> lo2, m2;
    lo2.reserve(lo.size() * 2);
    m2.reserve(lo.size() * 2);
    for (size_t i = 0; i < lo.size(); ++i) {
      const uint64_t h = m[i] >> 1;
      lo2.push_back(lo[i]);
      m2.push_back(h);
      lo2.push_back(lo[i] + h);
      m2.push_back(m[i] - h);
    }
    lo.swap(lo2);
    m.swap(m2);
  }
  std::vector<uint32_t> out(lo.size() + 1);
  for (size_t i = 0; i < lo.size(); ++i) out[i] = (uint32_t)lo[i];
  out[lo.size()] = (uint32_t)n;
  return out;
}

// The per-chunk metadata of one row shape, built on the host and uploaded
// once: {jb0, nblk, le, 0, lo[jb0 .. jb0 + nblk]} per chunk k of the row
// (blocks starting in [k*CH, (k+1)*CH); le = end of the last one).
qfb_status sb_shape(qfb_ctx* ctx, uint64_t n, uint32_t depth, const uint32_t** meta, uint32_t* nch) {
  for (const auto& kv : ctx->sb_shapes)
    if (kv.first == n) {
      *meta = kv.second.meta;
      *nch = kv.second.nch;
      return QFB_OK;
    }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(ctx->stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
    return fail(QFB_ERR_UNSUPPORTED, "backward: row length %llu first seen during a stream capture: run the "
                "call once eagerly (or qfb_fq_bwd_reserve) before capturing", (unsigned long long)n);
  const uint32_t L = depth - (uint32_t)kSbBlockLog;
  const std::vector<uint32_t> lo = tree_starts(n, L);
  const uint32_t NB = 1u << L;
  const uint32_t k_n = (uint32_t)((n + kSbChunk - 1) / kSbChunk);
  std::vector<uint32_t> tab((size_t)k_n * kSbMetaWords, 0u);
  for (uint32_t k = 0; k < k_n; ++k) {
    const uint32_t c0 = k * (uint32_t)kSbChunk;
    const uint32_t c1 = (uint32_t)std::min<uint64_t>(c0 + (uint64_t)kSbChunk, n);
    const uint32_t jb0 = (uint32_t)(std::lower_bound(lo.begin(), lo.begin() + NB, c0) - lo.begin());
    const uint32_t jb1 = (uint32_t)(std::lower_bound(lo.begin(), lo.begin() + NB, c1) - lo.begin());
    const uint32_t nblk = jb1 - jb0;
    if (nblk > (uint32_t)kSbMaxBlocks || (nblk && lo[jb1] - c0 > (uint32_t)kSbWin))
      return fail(QFB_ERR_UNSUPPORTED, "backward: block layout of a %llu-element row exceeds the chunk bounds",
                  (unsigned long long)n);
    uint32_t* e = tab.data() + (size_t)k * kSbMetaWords;
    e[0] = jb0;
    e[1] = nblk;
    e[2] = nblk ? lo[jb1] : c1;
    for (uint32_t i = 0; i <= nblk; ++i) e[4 + i] = lo[jb0 + i];
  }
  qfb_ctx::SbShape sh;
  QFB_CUDA(cudaMalloc(&sh.meta, tab.size() * sizeof(uint32_t)));
  QFB_CUDA(cudaMemcpy(sh.meta, tab.data(), tab.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
  sh.nch = k_n;
  ctx->sb_shapes.emplace_back(n, sh);
  *meta = sh.meta;
  *nch = k_n;
  return QFB_OK;
}

// Switch a plan to the streaming kernel: block partials (part_log = D - 4),
// chunks instead of tiles.
qfb_status sb_plan(qfb_ctx* ctx, BwdPlan& p) {
  BwdDesc& d = p.d;
  const uint32_t* meta = nullptr;
  uint32_t nch = 0;
  if (qfb_status st = sb_shape(ctx, d.inner, d.depth, &meta, &nch)) return st;
  d.sb_meta = meta;
  d.sb_nch = nch;
  d.sb_nch_div = make_fastdiv(nch);
  d.part_log = d.depth - (uint32_t)kSbBlockLog;
  const uint64_t segs = (uint64_t)d.outer * d.chans;
  p.tiles = segs * nch;
  p.f64_need = segs << d.part_log;
  if (p.tiles >= (1ull << 31)) return fail(QFB_ERR_UNSUPPORTED, "too many chunks");
  return QFB_OK;
}

// Plans of a table, switched to the streaming kernel when every entry is
// eligible (one launch for the whole table, as for the tile kernel).
qfb_status plan_bwd_table(qfb_ctx* ctx, int dtype, const qfb_bwd_desc* table, int32_t n,
                          std::vector<BwdPlan>& plans, bool* stream, bool* warp_part) {
  plans.assign((size_t)n, BwdPlan{});
  for (int32_t i = 0; i < n; ++i)
    if (qfb_status st = plan_bwd(table[i], plans[i], dtype)) return st;
  bool all = ctx->bwd_impl == 2 && n > 0 && ctx->sb_blocks_per_sm[dtype] > 0;
  for (int32_t i = 0; i < n && all; ++i) all = sb_eligible(plans[i], dtype);
  *stream = all;
  if (all)
    for (auto& p : plans)
      if (qfb_status st = sb_plan(ctx, p)) return st;
  // tile kernel: consumer-side warp sums when every row has full 256-group
  // tiles (g == kBwdGroupsLog)
  *warp_part = false;
  if (!all && ctx->bwd_impl == 0) {
    bool wp = n > 0;
    for (int32_t i = 0; i < n && wp; ++i) wp = plans[i].d.g == (uint32_t)kBwdGroupsLog;
    *warp_part = wp;
  }
  return QFB_OK;
}

}  // namespace

qfb_status qfb_fq_bwd_reserve(qfb_ctx* ctx, qfb_dtype dtype, const qfb_bwd_desc* table, int32_t n) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = check_dtype(dtype)) return st;
  if (n < 0 || (n > 0 && !table)) return fail(QFB_ERR_VALUE, "fq_bwd_reserve: bad table");
  size_t need = 1, f64 = 0;
  int32_t cnt = 0;
  uint64_t tiles = 0;
  std::vector<BwdPlan> plans;
  bool stream = false, warp_part = false;
  DeviceGuard g0(ctx->device);
  if (qfb_status st = plan_bwd_table(ctx, dtype, table, n, plans, &stream, &warp_part)) return st;
  for (int32_t i = 0; i < n; ++i) {
    const BwdPlan& p = plans[(size_t)i];
    // the same batching as qfb_fq_bwd_multi: the largest batch sizes it
    if (cnt == kMaxBwdDesc || (cnt > 0 && tiles + p.tiles >= (1ull << 31))) {
      need = std::max(need, f64);
      f64 = 0;
      cnt = 0;
      tiles = 0;
    }
    f64 += p.f64_need;
    tiles += p.tiles;
    ++cnt;
  }
  need = std::max(need, f64);
  DeviceGuard g(ctx->device);
  return grow(ctx, ctx->ws_f64, need * 8, false);
}

qfb_status qfb_fq_bwd_multi(qfb_ctx* ctx, qfb_dtype dtype, const qfb_bwd_desc* table, int32_t n) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = check_dtype(dtype)) return st;
  if (n < 0 || (n > 0 && !table)) return fail(QFB_ERR_VALUE, "fq_bwd_multi: bad table");
  DeviceGuard g(ctx->device);
  std::vector<BwdPlan> plans;
  bool stream = false, warp_part = false;
  if (qfb_status st = plan_bwd_table(ctx, dtype, table, n, plans, &stream, &warp_part)) return st;
  // an asynchronous finisher still reading the partials workspace
  if (qfb_status st = qfb_ctx_join(ctx)) return st;
  int32_t i = 0;
  while (i < n) {
    // Batch up to kMaxBwdDesc entries; each gets its own workspace slice.
    int32_t cnt = 0;
    size_t f64 = 0, u32 = 0;
    uint64_t tiles = 0;
    while (i + cnt < n && cnt < kMaxBwdDesc) {
      const BwdPlan& p = plans[i + cnt];
      if (cnt > 0 && tiles + p.tiles >= (1ull << 31)) break;
      f64 += p.f64_need;
      u32 += p.u32_need;
      tiles += p.tiles;
      ++cnt;
    }
    if (qfb_status st = grow(ctx, ctx->ws_f64, std::max<size_t>(f64, 1) * 8, false)) return st;
    BwdBatch b;
    std::memset(&b, 0, sizeof b);
    double* fp = static_cast<double*>(ctx->ws_f64.p);
    uint64_t tb = 0;
    for (int32_t k = 0; k < cnt; ++k) {
      BwdDesc d = plans[i + k].d;
      const uint64_t segs = (uint64_t)d.outer * d.chans;
      const uint64_t tps = 1ull << d.part_log;
      d.partials = fp;
      fp += segs * tps;

      b.d[k] = d;
      b.tile_begin[k] = (uint32_t)tb;
      tb += plans[i + k].tiles;
    }
    b.n = cnt;
    b.tile_begin[cnt] = (uint32_t)tb;
    b.warp_part = warp_part ? 1u : 0u;
    b.layout = ctx->bwd_layout | ctx->bwd_order | ((dtype == QFB_F16 && ctx->bwd_half_fp32) ? kBwdLayoutHalfF32 : 0u);
    if (stream) {
      const int grid = ctx->sm_count * ctx->sb_blocks_per_sm[dtype];
      cudaError_t e = launch_sbwd(dtype, sb_stages(dtype), b, grid, ctx->stream);
      if (e != cudaSuccess) return cuda_fail(e, "sbwd_kernel launch");
      ctx->launches += 2;  // main pass + finisher
      i += cnt;
      continue;
    }
    // ring sized from the largest tile of the batch (node size bound)
    uint32_t max_tile = 1;
    for (int32_t k = 0; k < cnt; ++k) {
      const uint64_t span = 1ull << b.d[k].tps_log;
      max_tile = std::max<uint32_t>(max_tile, (uint32_t)((b.d[k].inner + span - 1) / span));
    }
    size_t smem = 0;
    bwd_ring_size(dtype, max_tile, &b.stage_elems, &b.nstages, &smem);
    // cached: keeps steady-state launches free of runtime queries (graph capture)
    int per_sm = 0;
    const size_t key = (smem * 2 + (warp_part ? 1 : 0)) * 128 + b.layout;
    for (const auto& kv : ctx->bwd_occ[dtype])
      if (kv.first == key) per_sm = kv.second;
    if (per_sm == 0) {
      if (bwd_occupancy_smem(dtype, smem, &per_sm, warp_part, b.layout) != cudaSuccess || per_sm < 1) per_sm = 1;
      ctx->bwd_occ[dtype].emplace_back(key, per_sm);
    }
    const int grid = ctx->sm_count * per_sm;
    // a later batch reuses the partials: join the previous batch's finisher
    if (qfb_status st = qfb_ctx_join(ctx)) return st;
    const bool async = ctx->async_finish && ctx->side;
    cudaError_t e = launch_bwd(dtype, b, grid, ctx->stream, ctx->main_pass_event, async ? ctx->side : nullptr,
                               ctx->ev_fork);
    if (e == cudaSuccess && async) {
      e = cudaEventRecord(ctx->ev_join, ctx->side);
      ctx->side_pending = true;
    }
    if (e != cudaSuccess) return cuda_fail(e, "bwd_kernel launch");
    ctx->launches += 2;  // main pass + finisher
    i += cnt;
  }
  return QFB_OK;
}

qfb_status qfb_fq_bwd(qfb_ctx* ctx, qfb_dtype dtype, const void* x, const void* up, void* dx,
                      int64_t outer, int64_t channels, int64_t inner, const double* scale64,
                      const double* chain, int32_t q_max, double* d_log_s, int32_t accumulate) {
  qfb_bwd_desc t{x, up, dx, scale64, chain, d_log_s, outer, channels, inner, q_max, accumulate, 0};
  return qfb_fq_bwd_multi(ctx, dtype, &t, 1);
}

// ------------------------------------------------ host-level ops ---
namespace {

qfb_status h2d(qfb_ctx* ctx, DevBuf& b, const void* src, size_t bytes) {
  if (qfb_status st = grow(ctx, b, bytes, false)) return st;
  QFB_CUDA(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return QFB_OK;
}

}  // namespace

qfb_status qfb_fake_quantize_host(qfb_ctx* ctx, qfb_precision prec, const float* x, float* y,
                                  int64_t outer, int64_t channels, int64_t inner,
                                  const double* s, const qfb_quant_config* cfg) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = qfb_quant_config_validate(cfg)) return st;
  if (qfb_status st = check_dims(outer, channels, inner, "fake_quantize")) return st;
  if (!x || !y || !s) return fail(QFB_ERR_VALUE, "fake_quantize: null pointer");
  std::vector<float> sf((size_t)channels);
  if (qfb_status st = qfb_cast_scales_f32(s, channels, sf.data())) return st;
  const size_t bytes = (size_t)(outer * channels * inner) * sizeof(float);
  DeviceGuard g(ctx->device);
  if (qfb_status st = h2d(ctx, ctx->host_io[0], x, bytes)) return st;
  if (qfb_status st = h2d(ctx, ctx->host_io[2], sf.data(), sf.size() * sizeof(float))) return st;
  if (qfb_status st = grow(ctx, ctx->host_io[1], bytes, false)) return st;
  const uint32_t flags = prec == QFB_PREC_HALF ? QFB_FLAG_HALF_GRID : 0u;
  if (qfb_status st = qfb_fq_fwd(ctx, QFB_F32, ctx->host_io[0].p, ctx->host_io[1].p, outer,
                                 channels, inner, static_cast<const float*>(ctx->host_io[2].p),
                                 qfb_q_max(cfg), flags))
    return st;
  QFB_CUDA(cudaMemcpyAsync(y, ctx->host_io[1].p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  return qfb_ctx_sync(ctx);
}

qfb_status qfb_int8_codes_host(qfb_ctx* ctx, const float* x, int8_t* codes, int64_t outer,
                               int64_t channels, int64_t inner, const double* s,
                               const qfb_quant_config* cfg) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = qfb_quant_config_validate(cfg)) return st;
  if (qfb_status st = check_dims(outer, channels, inner, "int8_codes")) return st;
  if (!x || !codes || !s) return fail(QFB_ERR_VALUE, "int8_codes: null pointer");
  std::vector<float> sf((size_t)channels);
  if (qfb_status st = qfb_cast_scales_f32(s, channels, sf.data())) return st;
  const size_t n = (size_t)(outer * channels * inner);
  DeviceGuard g(ctx->device);
  if (qfb_status st = h2d(ctx, ctx->host_io[0], x, n * sizeof(float))) return st;
  if (qfb_status st = h2d(ctx, ctx->host_io[2], sf.data(), sf.size() * sizeof(float))) return st;
  if (qfb_status st = grow(ctx, ctx->host_io[1], n, false)) return st;
  if (qfb_status st = qfb_int8_codes(ctx, QFB_F32, ctx->host_io[0].p,
                                     static_cast<int8_t*>(ctx->host_io[1].p), outer, channels,
                                     inner, static_cast<const float*>(ctx->host_io[2].p),
                                     qfb_q_max(cfg)))
    return st;
  QFB_CUDA(cudaMemcpyAsync(codes, ctx->host_io[1].p, n, cudaMemcpyDeviceToHost, ctx->stream));
  return qfb_ctx_sync(ctx);
}

qfb_status qfb_fake_quantize_backward_host(qfb_ctx* ctx, qfb_precision prec, const float* x,
                                           const float* up, float* dx, int64_t outer,
                                           int64_t channels, int64_t inner,
                                           const double* log_s, const qfb_quant_config* cfg,
                                           double* d_log_s, int32_t accumulate) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = qfb_quant_config_validate(cfg)) return st;
  if (qfb_status st = check_dims(outer, channels, inner, "fake_quantize_backward")) return st;
  if (!x || !up || !log_s || !d_log_s) return fail(QFB_ERR_VALUE, "fake_quantize_backward: null pointer");
  std::vector<double> fac((size_t)channels * 3);
  double* s64 = fac.data();
  double* chain = fac.data() + channels;
  double* acc = fac.data() + 2 * channels;
  if (qfb_status st = qfb_scale_grad_factors(log_s, channels, cfg, prec, s64, chain)) return st;
  for (int64_t c = 0; c < channels; ++c) acc[c] = accumulate ? d_log_s[c] : 0.0;
  const size_t bytes = (size_t)(outer * channels * inner) * sizeof(float);
  DeviceGuard g(ctx->device);
  if (qfb_status st = h2d(ctx, ctx->host_io[0], x, bytes)) return st;
  if (qfb_status st = h2d(ctx, ctx->host_io[1], up, bytes)) return st;
  if (qfb_status st = h2d(ctx, ctx->host_io[3], fac.data(), fac.size() * sizeof(double))) return st;
  if (dx)
    if (qfb_status st = grow(ctx, ctx->host_io[4], bytes, false)) return st;
  const double* dfac = static_cast<const double*>(ctx->host_io[3].p);
  double* dacc = static_cast<double*>(ctx->host_io[3].p) + 2 * channels;
  if (qfb_status st = qfb_fq_bwd(ctx, QFB_F32, ctx->host_io[0].p, ctx->host_io[1].p,
                                 dx ? ctx->host_io[4].p : nullptr, outer, channels, inner, dfac,
                                 dfac + channels, qfb_q_max(cfg), dacc, accumulate))
    return st;
  if (qfb_status st = qfb_ctx_join(ctx)) return st;  // d_log_s complete (async finisher)
  if (dx) QFB_CUDA(cudaMemcpyAsync(dx, ctx->host_io[4].p, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  QFB_CUDA(cudaMemcpyAsync(d_log_s, dacc, (size_t)channels * sizeof(double),
                           cudaMemcpyDeviceToHost, ctx->stream));
  return qfb_ctx_sync(ctx);
}

namespace {

// A few host<->device copies on one stream as one submission
// (cudaMemcpyBatchAsync, stream-ordered sources); QFB_BATCH_COPY=0 falls
// back to one cudaMemcpyAsync per buffer.
qfb_status copy_batch(void** dst, void** src, size_t* sz, size_t n, cudaStream_t st) {
  static const bool batch = [] {
    const char* e = getenv("QFB_BATCH_COPY");
    return !(e && e[0] == '0');
  }();
  // merge runs contiguous on both sides into one copy: each DMA copy costs
  // ~10-20 us of engine overhead when both directions run
  // (tools/copy_probe.py); QFB_MERGE_COPY=0 disables (A/B)
  static const bool merge = [] {
    const char* e = getenv("QFB_MERGE_COPY");
    return !(e && e[0] == '0');
  }();
  if (merge && n > 1) {
    size_t m = 0;
    for (size_t i = 0; i < n; ++i) {
      if (m > 0 && static_cast<char*>(dst[m - 1]) + sz[m - 1] == dst[i] &&
          static_cast<char*>(src[m - 1]) + sz[m - 1] == src[i]) {
        sz[m - 1] += sz[i];
        continue;
      }
      dst[m] = dst[i];
      src[m] = src[i];
      sz[m] = sz[i];
      ++m;
    }
    n = m;
  }
  if (n == 0) return QFB_OK;
  if (!batch || n == 1) {
    for (size_t i = 0; i < n; ++i) QFB_CUDA(cudaMemcpyAsync(dst[i], src[i], sz[i], cudaMemcpyDefault, st));
    return QFB_OK;
  }
  cudaMemcpyAttributes attr{};
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  size_t idx = 0, fail = 0;
  QFB_CUDA(cudaMemcpyBatchAsync(dst, src, sz, n, &attr, &idx, 1, &fail, st));
  return QFB_OK;
}

}  // namespace

qfb_status qfb_quant_pass_host_submit(qfb_ctx* ctx, qfb_precision prec, const qfb_host_point* pts,
                                      int32_t n, const qfb_quant_config* cfg, int32_t slot) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (qfb_status st = qfb_quant_config_validate(cfg)) return st;
  if (n < 0 || (n > 0 && !pts)) return fail(QFB_ERR_VALUE, "quant_pass_host: bad table");
  if (slot < 0 || slot > 1) return fail(QFB_ERR_VALUE, "quant_pass_host: slot must be 0 or 1");
  auto& sl = ctx->slots[slot];
  if (sl.busy) return fail(QFB_ERR_VALUE, "quant_pass_host: slot %d still in flight (wait first)", slot);
  sl.grads.clear();
  sl.grad_len.clear();
  if (n == 0) return QFB_OK;
  const int32_t q = qfb_q_max(cfg);
  // ---- validate everything and build the parameter block on the host
  // layout per point k: [s32 (2*C floats padded)...] then doubles; keep it
  // simple: one double block {s64|chain|acc} x 2 consumers, one float block
  std::vector<size_t> foff((size_t)n), doff((size_t)n);
  size_t fcount = 0, dcount = 0;
  for (int32_t i = 0; i < n; ++i) {
    const qfb_host_point& p = pts[i];
    if (qfb_status st = check_dims(p.outer, p.channels, p.inner, "quant_pass_host")) return st;
    if (!p.x || p.n_out < 1 || p.n_out > 2) return fail(QFB_ERR_VALUE, "quant_pass_host: point %d", i);
    for (int k = 0; k < p.n_out; ++k) {
      if (p.y[k] && !p.s[k]) return fail(QFB_ERR_VALUE, "quant_pass_host: point %d needs scales", i);
      if (p.log_s[k] && (!p.up[k] || !p.d_log_s[k]))
        return fail(QFB_ERR_VALUE, "quant_pass_host: point %d backward needs up/d_log_s", i);
    }
    foff[i] = fcount;
    fcount += (size_t)(2 * p.channels + 4);   // 16-byte aligned float slots
    fcount = (fcount + 3) & ~size_t(3);
    doff[i] = dcount;
    dcount += (size_t)(6 * p.channels);
  }
  std::vector<float> fblk(fcount, 0.0f);
  std::vector<double> dblk(dcount, 0.0);
  for (int32_t i = 0; i < n; ++i) {
    const qfb_host_point& p = pts[i];
    for (int k = 0; k < p.n_out; ++k) {
      if (p.y[k])
        if (qfb_status st = qfb_cast_scales_f32(p.s[k], p.channels, fblk.data() + foff[i] + k * p.channels))
          return st;
      if (p.log_s[k]) {
        double* b = dblk.data() + doff[i] + (size_t)k * 3 * p.channels;
        if (qfb_status st = qfb_scale_grad_factors(p.log_s[k], p.channels, cfg, prec, b, b + p.channels))
          return st;
      }
    }
  }
  DeviceGuard g(ctx->device);
  if (!ctx->s_in) {
    QFB_CUDA(cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking));
    QFB_CUDA(cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking));
  }
  if (!sl.done) QFB_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
  while ((int32_t)sl.ev.size() < 2 * n + 1) {
    cudaEvent_t e;
    QFB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sl.ev.push_back(e);
  }
  const size_t pbytes = fcount * sizeof(float) + dcount * sizeof(double);
  if (qfb_status st = grow(ctx, sl.params, pbytes, false)) return st;
  float* dF = static_cast<float*>(sl.params.p);
  double* dD = reinterpret_cast<double*>(static_cast<char*>(sl.params.p) + fcount * sizeof(float));
  // Pinned staging: a copy from/to pageable memory is synchronous for the
  // issuing thread and would serialize the pipeline. One extra slot at the
  // end receives the status word.
  if (sl.pinned_bytes < pbytes + 16) {
    if (sl.pinned) QFB_CUDA(cudaFreeHost(sl.pinned));
    sl.pinned = nullptr;
    sl.pinned_bytes = 0;
    QFB_CUDA(cudaMallocHost(&sl.pinned, pbytes + 16));
    sl.pinned_bytes = pbytes + 16;
  }
  float* hF = static_cast<float*>(sl.pinned);
  double* hD = reinterpret_cast<double*>(static_cast<char*>(sl.pinned) + fcount * sizeof(float));
  sl.h_status = reinterpret_cast<uint32_t*>(static_cast<char*>(sl.pinned) + pbytes);
  sl.grad_base = hD;
  std::memcpy(hF, fblk.data(), fcount * sizeof(float));
  std::memcpy(hD, dblk.data(), dcount * sizeof(double));
  // QFB_PASS_TIMING=1: stage timestamps of this pass on stderr (diagnostics)
  static const bool timing = [] {
    const char* e = getenv("QFB_PASS_TIMING");
    return e && e[0] == '1';
  }();
  cudaEvent_t te[4] = {nullptr, nullptr, nullptr, nullptr};
  if (timing)
    for (auto& e : te) QFB_CUDA(cudaEventCreate(&e));
  // all streams start after prior work on the context stream
  QFB_CUDA(cudaEventRecord(sl.ev[2 * n], ctx->stream));
  QFB_CUDA(cudaStreamWaitEvent(ctx->s_in, sl.ev[2 * n], 0));
  if (timing) QFB_CUDA(cudaEventRecord(te[0], ctx->s_in));
  QFB_CUDA(cudaMemcpyAsync(dF, hF, pbytes, cudaMemcpyHostToDevice, ctx->s_in));
  // per point: x, up[2], y[2], dx[2] inside the two arenas (copy order;
  // 16-byte aligned offsets)
  sl.ptr.assign((size_t)n * 7, nullptr);
  {
    std::vector<size_t> off((size_t)n * 7, 0);
    size_t in_b = 0, out_b = 0;
    auto take = [](size_t& cur, size_t bytes) {
      const size_t o = cur;
      cur += (bytes + 15) & ~size_t(15);
      return o;
    };
    for (int32_t i = 0; i < n; ++i) {
      const qfb_host_point& p = pts[i];
      const size_t bytes = (size_t)(p.outer * p.channels * p.inner) * sizeof(float);
      off[(size_t)i * 7] = take(in_b, bytes);
      for (int k = 0; k < p.n_out; ++k)
        if (p.log_s[k]) off[(size_t)i * 7 + 1 + k] = take(in_b, bytes);
      for (int k = 0; k < p.n_out; ++k) {
        if (p.y[k]) off[(size_t)i * 7 + 3 + k] = take(out_b, bytes);
        if (p.log_s[k] && p.dx[k]) off[(size_t)i * 7 + 5 + k] = take(out_b, bytes);
      }
    }
    if (qfb_status st = grow(ctx, sl.in_arena, std::max<size_t>(in_b, 16), false)) return st;
    if (qfb_status st = grow(ctx, sl.out_arena, std::max<size_t>(out_b, 16), false)) return st;
    for (int32_t i = 0; i < n; ++i) {
      const qfb_host_point& p = pts[i];
      void** P = &sl.ptr[(size_t)i * 7];
      P[0] = static_cast<char*>(sl.in_arena.p) + off[(size_t)i * 7];
      for (int k = 0; k < p.n_out; ++k) {
        if (p.log_s[k]) P[1 + k] = static_cast<char*>(sl.in_arena.p) + off[(size_t)i * 7 + 1 + k];
        if (p.y[k]) P[3 + k] = static_cast<char*>(sl.out_arena.p) + off[(size_t)i * 7 + 3 + k];
        if (p.log_s[k] && p.dx[k]) P[5 + k] = static_cast<char*>(sl.out_arena.p) + off[(size_t)i * 7 + 5 + k];
      }
    }
  }
  // ---- pipeline: H2D (s_in) -> kernels (ctx->stream) -> D2H (s_out), in
  // groups of points: each group's inputs go as one batched submission, its
  // kernels wait for that submission, its outputs go back as one batched
  // submission (per-copy overhead is ~10-20 us when both directions run;
  // smaller groups pipeline better, QFB_PASS_GROUP tunes the size)
  static const int32_t group_pts = [] {
    const char* e = getenv("QFB_PASS_GROUP");
    const int v = e ? atoi(e) : 0;
    return v > 0 ? v : 1;  // measured: 1 point per group is best (7.40 ms/frame vs 7.42, 7.73 for 2, 3)
  }();
  const uint32_t flags = prec == QFB_PREC_HALF ? QFB_FLAG_HALF_GRID : 0u;
  // this slot's kernels latch non-finite results into the slot's own status
  // word (restored on every exit), copied down and cleared on s_out below,
  // so a non-finite value is reported by this slot's wait and no other's
  uint32_t* const slot_status = ctx->d_status + 1 + slot;
  struct StatusScope {
    qfb_ctx* c;
    uint32_t* prev;
    ~StatusScope() { c->cur_status = prev; }
  } status_scope{ctx, ctx->cur_status};
  ctx->cur_status = slot_status;
  std::vector<void*> cdst, csrc;
  std::vector<size_t> csz;
  // groups of points by input bytes (default 80 MB: 4 groups per DPVO
  // frame): with host buffers laid out in copy order, each group's copies
  // merge into one per direction. Measured (`profiles/r02_aq_*`): 141 ->
  // 151 frames/s end to end, 98 % of the concurrent H2D + D2H ceiling; the
  // per-point pipeline with merging alone: 142. QFB_PASS_GROUP_MB=0 restores
  // per-point groups (QFB_PASS_GROUP points each).
  static const double group_mb = [] {
    const char* e = getenv("QFB_PASS_GROUP_MB");
    return e ? atof(e) : 80.0;
  }();
  for (int32_t g0 = 0, g1 = 0; g0 < n; g0 = g1) {
    g1 = std::min(n, g0 + group_pts);
    if (group_mb > 0.0) {
      double mb = 0.0;
      g1 = g0;
      while (g1 < n && (g1 == g0 || mb < group_mb)) {
        const qfb_host_point& p = pts[g1];
        int nin = 1;
        for (int k = 0; k < p.n_out; ++k) nin += p.log_s[k] ? 1 : 0;
        mb += (double)(p.outer * p.channels * p.inner) * sizeof(float) * nin / 1e6;
        ++g1;
      }
    }
    cdst.clear();
    csrc.clear();
    csz.clear();
    for (int32_t i = g0; i < g1; ++i) {
      const qfb_host_point& p = pts[i];
      const size_t bytes = (size_t)(p.outer * p.channels * p.inner) * sizeof(float);
      void* const* B = &sl.ptr[(size_t)i * 7];
      cdst.push_back(B[0]), csrc.push_back(const_cast<float*>(p.x)), csz.push_back(bytes);
      for (int k = 0; k < p.n_out; ++k)
        if (p.log_s[k])
          cdst.push_back(B[1 + k]), csrc.push_back(const_cast<float*>(p.up[k])), csz.push_back(bytes);
    }
    if (qfb_status st = copy_batch(cdst.data(), csrc.data(), csz.data(), cdst.size(), ctx->s_in)) return st;
    QFB_CUDA(cudaEventRecord(sl.ev[2 * g0], ctx->s_in));
    QFB_CUDA(cudaStreamWaitEvent(ctx->stream, sl.ev[2 * g0], 0));
    for (int32_t i = g0; i < g1; ++i) {
      const qfb_host_point& p = pts[i];
      void* const* B = &sl.ptr[(size_t)i * 7];
      // forward: one launch for all consumers of this tensor
      bool any_y = false;
      qfb_fq_desc fd{};
      fd.x = B[0];
      fd.outer = p.outer;
      fd.channels = p.channels;
      fd.inner = p.inner;
      fd.q_max = q;
      fd.flags = flags;
      int no = 0;
      for (int k = 0; k < p.n_out; ++k) {
        if (!p.y[k]) continue;
        fd.y[no] = B[3 + k];
        fd.scale[no] = dF + foff[i] + k * p.channels;
        ++no;
        any_y = true;
      }
      fd.n_out = no;
      if (any_y)
        if (qfb_status st = qfb_fq_fwd_multi(ctx, QFB_F32, &fd, 1)) return st;
      // backward per consumer
      qfb_bwd_desc bd[2];
      int nb = 0;
      for (int k = 0; k < p.n_out; ++k) {
        if (!p.log_s[k]) continue;
        const double* f = dD + doff[i] + (size_t)k * 3 * p.channels;
        bd[nb] = qfb_bwd_desc{B[0], B[1 + k], p.dx[k] ? B[5 + k] : nullptr, f, f + p.channels,
                              const_cast<double*>(f + 2 * p.channels), p.outer, p.channels, p.inner, q, 0, 0};
        ++nb;
      }
      if (nb) {
        if (qfb_status st = qfb_fq_bwd_multi(ctx, QFB_F32, bd, nb)) return st;
        if (qfb_status st = qfb_ctx_join(ctx)) return st;  // d_log_s complete (async finisher)
      }
    }
    QFB_CUDA(cudaEventRecord(sl.ev[2 * g0 + 1], ctx->stream));
    QFB_CUDA(cudaStreamWaitEvent(ctx->s_out, sl.ev[2 * g0 + 1], 0));
    cdst.clear();
    csrc.clear();
    csz.clear();
    for (int32_t i = g0; i < g1; ++i) {
      const qfb_host_point& p = pts[i];
      const size_t bytes = (size_t)(p.outer * p.channels * p.inner) * sizeof(float);
      void* const* B = &sl.ptr[(size_t)i * 7];
      for (int k = 0; k < p.n_out; ++k) {
        if (p.y[k]) cdst.push_back(p.y[k]), csrc.push_back(B[3 + k]), csz.push_back(bytes);
        if (p.log_s[k] && p.dx[k]) cdst.push_back(p.dx[k]), csrc.push_back(B[5 + k]), csz.push_back(bytes);
      }
    }
    if (qfb_status st = copy_batch(cdst.data(), csrc.data(), csz.data(), cdst.size(), ctx->s_out)) return st;
  }
  // all scale gradients in one copy (they sit in the parameter block)
  QFB_CUDA(cudaMemcpyAsync(hD, dD, dcount * sizeof(double), cudaMemcpyDeviceToHost, ctx->s_out));
  if (timing) {
    QFB_CUDA(cudaEventRecord(te[1], ctx->s_in));
    QFB_CUDA(cudaEventRecord(te[2], ctx->stream));
    QFB_CUDA(cudaEventRecord(te[3], ctx->s_out));
  }
  // the status word of this pass's kernels rides down with the gradients
  QFB_CUDA(cudaEventRecord(sl.ev[2 * n], ctx->stream));
  QFB_CUDA(cudaStreamWaitEvent(ctx->s_out, sl.ev[2 * n], 0));
  QFB_CUDA(cudaMemcpyAsync(sl.h_status, slot_status, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->s_out));
  QFB_CUDA(cudaMemsetAsync(slot_status, 0, sizeof(uint32_t), ctx->s_out));
  QFB_CUDA(cudaEventRecord(sl.done, ctx->s_out));
  for (int32_t i = 0; i < n; ++i) {
    const qfb_host_point& p = pts[i];
    for (int k = 0; k < p.n_out; ++k)
      if (p.log_s[k]) {
        sl.grads.emplace_back(p.d_log_s[k], doff[i] + (size_t)k * 3 * p.channels + 2 * p.channels);
        sl.grad_len.push_back(p.channels);
      }
  }
  sl.busy = true;
  if (timing) {
    QFB_CUDA(cudaEventSynchronize(te[3]));
    float ms[3];
    for (int k = 0; k < 3; ++k) QFB_CUDA(cudaEventElapsedTime(&ms[k], te[0], te[k + 1]));
    fprintf(stderr, "quant_pass_host: h2d done %.3f ms, compute done %.3f ms, d2h done %.3f ms\n", ms[0], ms[1],
            ms[2]);
    for (auto& e : te) cudaEventDestroy(e);
  }
  return QFB_OK;
}

qfb_status qfb_quant_pass_host_wait(qfb_ctx* ctx, int32_t slot) {
  if (qfb_status st = check_ctx(ctx)) return st;
  if (slot < 0 || slot > 1) return fail(QFB_ERR_VALUE, "quant_pass_host: slot must be 0 or 1");
  auto& sl = ctx->slots[slot];
  if (!sl.busy) return QFB_OK;
  DeviceGuard g(ctx->device);
  sl.busy = false;
  QFB_CUDA(cudaEventSynchronize(sl.done));
  for (size_t i = 0; i < sl.grads.size(); ++i)
    std::memcpy(sl.grads[i].first, sl.grad_base + sl.grads[i].second, (size_t)sl.grad_len[i] * sizeof(double));
  // the slot's word was cleared on s_out after its copy (ordered before
  // `done`), so nothing is left to reset here
  if (*sl.h_status != 0)
    return fail(QFB_ERR_NONFINITE, "demote_half: non-finite value on the binary16 path (slot %d)", slot);
  return QFB_OK;
}

qfb_status qfb_quant_pass_host(qfb_ctx* ctx, qfb_precision prec, const qfb_host_point* pts, int32_t n,
                               const qfb_quant_config* cfg) {
  if (qfb_status st = qfb_quant_pass_host_wait(ctx, 0)) return st;
  if (qfb_status st = qfb_quant_pass_host_submit(ctx, prec, pts, n, cfg, 0)) return st;
  return qfb_quant_pass_host_wait(ctx, 0);
}

}  // extern "C"
