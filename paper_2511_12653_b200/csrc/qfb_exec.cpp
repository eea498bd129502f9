// qfb_exec.cpp — the execution plan: qf::run_quant_conv's quantization
// (exec.hpp:222-405) on the GPU, minus the convolution.
//
//   resolve pass   host libm resolve (bit-identical) -> device float[C_out+1]
//                  (exec.hpp:248-259), counted as one sweep
//   Fused          activation FQ (one kernel) + weight FQ (one kernel)
//                  (exec.hpp:344-381)
//   PerOperator    divide, clip, round, multiply as four kernels with float
//                  temporaries, for activations and weights (exec.hpp:276-342)
//   fault hook     fused path "throws" FusedPathError at fault_inject_layer;
//                  with fallback the layer reruns per-operator ON THE GPU and
//                  fell_back is recorded (exec.hpp:345-347, 383-393)
//   weight cache   frozen weights quantized once per plan (exec.hpp:59-60,
//                  261, 269-274)
//   counters       the reference's modeled sweep/byte rules
//                  (exec.hpp:199-216, :255, :289, :305, :322, :334, :361, :376)
// Both plans produce bit-identical outputs (tests/test_gpu_exec.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/qfb.h"

namespace {

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

qfb_status ensure(qfb_ctx* ctx, Buf& b, size_t bytes) {
  if (b.bytes >= bytes) return QFB_OK;
  if (b.p) {
    // earlier launches on the stream may still read it
    if (qfb_status st = qfb_ctx_sync(ctx)) return st;
    cudaFree(b.p);
  }
  b.p = nullptr;
  b.bytes = 0;
  if (cudaMalloc(&b.p, bytes) != cudaSuccess) return QFB_ERR_CUDA;
  b.bytes = bytes;
  return QFB_OK;
}

constexpr int64_t kF = 4;  // the reference's modeled element size (float)

void count(qfb_exec_trace* t, int64_t r, int64_t w) {
  t->pass_count += 1;
  t->bytes_read += r;
  t->bytes_written += w;
}

// exec.hpp:255 / :289-305 / :322-334 / :361 / :376
void model_resolve(qfb_exec_trace* t, int64_t c_out) { count(t, kF * (c_out + 1), kF * (c_out + 1)); }
void model_act(qfb_exec_trace* t, bool fused, int64_t na) {
  if (fused) {
    count(t, kF * na + 4, kF * na);
  } else {
    count(t, kF * na + 4, kF * na);  // divide (reads the scale)
    count(t, kF * na, kF * na);      // clip
    count(t, kF * na, kF * na);      // round
    count(t, kF * na + 4, kF * na);  // multiply (reads the scale)
  }
}
void model_weights(qfb_exec_trace* t, bool fused, int64_t nw, int64_t c_out) {
  if (fused) {
    count(t, kF * (nw + c_out), kF * nw);
  } else {
    count(t, kF * (nw + c_out), kF * nw);
    count(t, kF * nw, kF * nw);
    count(t, kF * nw, kF * nw);
    count(t, kF * (nw + c_out), kF * nw);
  }
}

}  // namespace

struct qfb_exec {
  qfb_ctx* ctx = nullptr;
  qfb_exec_plan plan{};
  qfb_exec_trace trace{};
  Buf scales;  // device float[c_out + 1]: weight scales then activation scale
  Buf tmp;     // per-operator temporaries: 3 * n floats
  std::map<int, Buf> cache;
};

extern "C" {

qfb_status qfb_exec_model_layer(const qfb_exec_plan* plan, int64_t n_act, int64_t c_out,
                                int64_t per, int32_t weights_cached, int32_t fused_fails,
                                qfb_exec_trace* delta) {
  if (!plan || !delta || n_act <= 0 || c_out <= 0 || per <= 0) return QFB_ERR_VALUE;
  std::memset(delta, 0, sizeof *delta);
  const bool fused = plan->mode == QFB_MODE_FUSED && !fused_fails;
  if (plan->mode == QFB_MODE_FUSED && fused_fails && !plan->fallback_enabled) return QFB_ERR_FUSED_PATH;
  model_resolve(delta, c_out);
  model_act(delta, fused, n_act);
  if (!weights_cached) model_weights(delta, fused, c_out * per, c_out);
  delta->fell_back = plan->mode == QFB_MODE_FUSED && fused_fails ? 1 : 0;
  delta->layers = 1;
  return QFB_OK;
}

qfb_status qfb_exec_create(qfb_ctx* ctx, const qfb_exec_plan* plan, qfb_exec** out) {
  if (!ctx || !plan || !out) return QFB_ERR_VALUE;
  if (plan->mode != QFB_MODE_FUSED && plan->mode != QFB_MODE_PER_OPERATOR) return QFB_ERR_VALUE;
  if (plan->policy != QFB_POLICY_FULL_ONLY && plan->policy != QFB_POLICY_HALF_ACTIVATIONS) return QFB_ERR_VALUE;
  qfb_exec* e = new qfb_exec();
  e->ctx = ctx;
  e->plan = *plan;
  *out = e;
  return QFB_OK;
}

qfb_status qfb_exec_destroy(qfb_exec* ex) {
  if (!ex) return QFB_OK;
  if (ex->ctx) qfb_ctx_sync(ex->ctx);
  if (ex->scales.p) cudaFree(ex->scales.p);
  if (ex->tmp.p) cudaFree(ex->tmp.p);
  for (auto& kv : ex->cache)
    if (kv.second.p) cudaFree(kv.second.p);
  delete ex;
  return QFB_OK;
}

qfb_status qfb_exec_trace_get(const qfb_exec* ex, qfb_exec_trace* out) {
  if (!ex || !out) return QFB_ERR_VALUE;
  *out = ex->trace;
  return QFB_OK;
}

qfb_status qfb_exec_trace_reset(qfb_exec* ex) {
  if (!ex) return QFB_ERR_VALUE;
  std::memset(&ex->trace, 0, sizeof ex->trace);
  return QFB_OK;
}

qfb_status qfb_exec_quant_layer(qfb_exec* ex, const qfb_quant_layer* L, const qfb_quant_config* cfg,
                                qfb_dtype dtype, const void* x, int64_t n_act, void* qa,
                                float* qw_buf, const float** qw) {
  if (!ex || !L || !cfg || !x || !qa || !qw) return QFB_ERR_VALUE;
  if (qfb_status st = qfb_quant_config_validate(cfg)) return st;
  if (n_act <= 0 || L->c_out <= 0 || L->per <= 0 || !L->weight || !L->log_w) return QFB_ERR_SHAPE;
  const bool half_acts = ex->plan.policy == QFB_POLICY_HALF_ACTIVATIONS;
  const qfb_precision act_mode = half_acts ? QFB_PREC_HALF : QFB_PREC_FULL;
  const int64_t c_out = L->c_out, nw = c_out * L->per;
  const bool use_cache = ex->plan.cache_weights && ex->cache.count(L->index) > 0;
  if (!use_cache && !qw_buf && !ex->plan.cache_weights) return QFB_ERR_VALUE;

  // The fused path's fault hook fires before any work (exec.hpp:345-347).
  bool fused = ex->plan.mode == QFB_MODE_FUSED;
  if (fused && ex->plan.fault_inject_layer == L->index) {
    if (!ex->plan.fallback_enabled) return QFB_ERR_FUSED_PATH;
    fused = false;
    ex->trace.fell_back = 1;
  }

  // Scale pass (exec.hpp:248-259): host libm, FP64 -> float.
  std::vector<double> sd((size_t)c_out + 1);
  if (qfb_status st = qfb_resolve_scales(L->log_w, c_out, cfg, QFB_PREC_FULL, sd.data())) return st;
  if (qfb_status st = qfb_resolve_scales(&L->log_a, 1, cfg, act_mode, sd.data() + c_out)) return st;
  std::vector<float> sf((size_t)c_out + 1);
  if (qfb_status st = qfb_cast_scales_f32(sd.data(), c_out + 1, sf.data())) return st;
  if (qfb_status st = ensure(ex->ctx, ex->scales, sf.size() * sizeof(float))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(qfb_ctx_stream(ex->ctx));
  if (cudaMemcpyAsync(ex->scales.p, sf.data(), sf.size() * sizeof(float), cudaMemcpyHostToDevice, s) !=
      cudaSuccess)
    return QFB_ERR_CUDA;
  model_resolve(&ex->trace, c_out);
  const float* d_sw = static_cast<const float*>(ex->scales.p);
  const float* d_sa = d_sw + c_out;
  const int32_t q = qfb_q_max(cfg);
  const uint32_t aflags = (half_acts && dtype == QFB_F32) ? QFB_FLAG_HALF_GRID : 0u;
  const int64_t before = qfb_ctx_launch_count(ex->ctx);

  // Activations: per-tensor scale s_a.
  if (fused) {
    if (qfb_status st = qfb_fq_fwd(ex->ctx, dtype, x, qa, 1, 1, n_act, d_sa, q, aflags)) return st;
  } else {
    const size_t need = (size_t)3 * std::max(n_act, use_cache ? 0 : nw) * sizeof(float);
    if (qfb_status st = ensure(ex->ctx, ex->tmp, need)) return st;
    ex->trace.peak_scratch_bytes = std::max<int64_t>(ex->trace.peak_scratch_bytes, (int64_t)need);
    if (qfb_status st = qfb_fq_fwd_perop(ex->ctx, dtype, x, qa, 1, 1, n_act, d_sa, q, aflags,
                                         static_cast<float*>(ex->tmp.p)))
      return st;
  }
  model_act(&ex->trace, fused, n_act);

  // Weights: per-channel along C_out, never demoted (exec.hpp:369-376).
  if (use_cache) {
    *qw = static_cast<const float*>(ex->cache[L->index].p);
  } else {
    float* dst = qw_buf;
    if (ex->plan.cache_weights) {
      Buf& b = ex->cache[L->index];
      if (qfb_status st = ensure(ex->ctx, b, (size_t)nw * sizeof(float))) return st;
      dst = static_cast<float*>(b.p);
    }
    if (fused) {
      if (qfb_status st = qfb_fq_fwd(ex->ctx, QFB_F32, L->weight, dst, 1, c_out, L->per, d_sw, q, 0u))
        return st;
    } else {
      if (qfb_status st = qfb_fq_fwd_perop(ex->ctx, QFB_F32, L->weight, dst, 1, c_out, L->per, d_sw, q,
                                           0u, static_cast<float*>(ex->tmp.p)))
        return st;
    }
    model_weights(&ex->trace, fused, nw, c_out);
    *qw = dst;
  }
  ex->trace.launches += qfb_ctx_launch_count(ex->ctx) - before;
  ex->trace.layers += 1;
  return QFB_OK;
}

}  // extern "C"
