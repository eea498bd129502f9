// subst_ops.cpp — the qfb side of the substitution (compiled with -Dqf=qfs,
// like subst.cpp): the qfb-backed overloads that the reference's
// fake_quantize / fake_quantize_backward call sites reach, and strong
// definitions of qfs::run_quant_conv and qfs::distill_loss that take the
// place of the headers' inline ones. Quantization, STE/LSQ backward and
// the distillation loss run on the GPU through libqfb (include/qfb.hpp,
// include/qfb.h); the convolution stays the reference's (out of scope,
// PAPER.md:142). Test infrastructure, not product code.
#include <algorithm>
#include <cmath>
#include <span>
#include <stdexcept>
#include <vector>

#include <cuda_runtime.h>

// The reference's own definitions of the two overridden functions (and of
// their callers, which would otherwise be emitted here calling them) are
// renamed out of the way in this TU only.
#define run_quant_conv dropin_unused_run_quant_conv
#define run_frontend dropin_unused_run_frontend
#define distill_loss dropin_unused_distill_loss
#define train_scales dropin_unused_train_scales
#include "quantfuse/distill.hpp"
#undef run_quant_conv
#undef run_frontend
#undef distill_loss
#undef train_scales

#include "qfb.hpp"
#include "dropin.h"

DropinCalls g_dropin_calls;

namespace {

qfb::Context& ctx() {
  static qfb::Context c(0);
  return c;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("dropin: ") + what + ": " + cudaGetErrorString(e));
}

// A device float buffer (test harness only; libqfb itself never allocates
// on the hot path, the caller owns device memory).
struct DevBuf {
  float* p = nullptr;
  explicit DevBuf(size_t n) { cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(float)), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

namespace qf {

// qfb throws qfb::ShapeError / ValueError / NonFiniteError / FusedPathError;
// the reference's callers catch qf:: types (e.g. train_scales catches
// NonFiniteError, distill.hpp:245), so rethrow under the reference's names.
template <class F>
auto translated(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const qfb::ShapeError& e) {
    throw ShapeError(e.what());
  } catch (const qfb::ValueError& e) {
    throw ValueError(e.what());
  } catch (const qfb::NonFiniteError& e) {
    throw NonFiniteError(e.what());
  } catch (const qfb::FusedPathError& e) {
    throw FusedPathError(e.what());
  }
}

Tensor qfb_fake_quantize(const Tensor& x, double s, const QuantConfig& cfg) {
  ++g_dropin_calls.fake_quantize;
  return translated([&] { return qfb::fake_quantize(ctx(), x, s, cfg); });
}

Tensor qfb_fake_quantize(const Tensor& x, std::span<const double> s, const QuantConfig& cfg) {
  ++g_dropin_calls.fake_quantize;
  return translated([&] { return qfb::fake_quantize(ctx(), x, s, cfg); });
}

FakeQuantGrad qfb_fake_quantize_backward(const Tensor& x, double log_s, const QuantConfig& cfg,
                                         const Tensor& upstream, Precision mode) {
  ++g_dropin_calls.fake_quantize_backward;
  auto g = translated([&] { return qfb::fake_quantize_backward(ctx(), x, log_s, cfg, upstream, mode); });
  return FakeQuantGrad{std::move(g.d_input), std::move(g.d_log_scale)};
}

FakeQuantGrad qfb_fake_quantize_backward(const Tensor& x, std::span<const double> log_s,
                                         const QuantConfig& cfg, const Tensor& upstream, Precision mode) {
  ++g_dropin_calls.fake_quantize_backward;
  auto g = translated([&] { return qfb::fake_quantize_backward(ctx(), x, log_s, cfg, upstream, mode); });
  return FakeQuantGrad{std::move(g.d_input), std::move(g.d_log_scale)};
}

// exec.hpp:222-405 with the scale pass and both quantization sweeps on the
// GPU (qfb_exec_quant_layer: Fused or PerOperator plan, injected fault ->
// per-operator fallback, HalfActivations store rounding), the weight cache
// kept where the reference keeps it (ctx.cached_weights), and the
// reference's conv on the quantized operands.
Tensor run_quant_conv(ExecutionContext& ectx, const ConvLayer& layer, int layer_idx, const Tensor& input) {
  ++g_dropin_calls.run_quant_conv;
  const bool half_acts = ectx.plan.policy == PrecisionPolicy::HalfActivations;
  const ConvEpilogue ep{layer.affine_scale, layer.affine_shift, layer.relu, half_acts};
  Tensor out;
  if (!layer.quantized) {
    out = conv2d(input, layer.weight, layer.stride, layer.padding, ep);
  } else {
    const int64_t c_out = layer.c_out();
    const int64_t na = input.numel(), nw = layer.weight.numel();
    const bool use_cache = ectx.plan.cache_weights && ectx.cached_weights.count(layer_idx) > 0;

    qfb_exec_plan plan{};
    plan.mode = ectx.plan.mode == ExecMode::Fused ? QFB_MODE_FUSED : QFB_MODE_PER_OPERATOR;
    plan.policy = half_acts ? QFB_POLICY_HALF_ACTIVATIONS : QFB_POLICY_FULL_ONLY;
    plan.fallback_enabled = ectx.plan.fallback_enabled ? 1 : 0;
    plan.cache_weights = 0;  // the cache lives in ectx.cached_weights, as in the reference
    plan.fault_inject_layer = ectx.plan.fault_inject_layer;
    qfb_exec* ex = nullptr;
    qfb::check(qfb_exec_create(ctx().get(), &plan, &ex));
    struct ExecGuard {
      qfb_exec* e;
      ~ExecGuard() { qfb_exec_destroy(e); }
    } guard{ex};

    DevBuf dx((size_t)na), dqa((size_t)na), dw((size_t)nw), dqw((size_t)nw);
    cuda_check(cudaMemcpy(dx.p, input.data.data(), na * sizeof(float), cudaMemcpyHostToDevice), "H2D x");
    cuda_check(cudaMemcpy(dw.p, layer.weight.data.data(), nw * sizeof(float), cudaMemcpyHostToDevice), "H2D w");
    const qfb_quant_config cfg = qfb::to_c(layer.qcfg);
    qfb_quant_layer ql{};
    ql.index = layer_idx;
    ql.weight = dw.p;
    ql.c_out = c_out;
    ql.per = nw / c_out;
    ql.log_w = layer.scales.log_w_scale.data();
    ql.log_a = layer.scales.log_a_scale;
    const float* qw = nullptr;
    const qfb_status st = qfb_exec_quant_layer(ex, &ql, &cfg, QFB_F32, dx.p, na, dqa.p, dqw.p, &qw);
    if (st == QFB_ERR_FUSED_PATH) throw FusedPathError(qfb_last_error());
    translated([&] {
      qfb::check(st);
      qfb::check(qfb_ctx_sync(ctx().get()));
    });
    qfb_exec_trace tr{};
    qfb::check(qfb_exec_trace_get(ex, &tr));
    if (tr.fell_back) ectx.trace.fell_back = true;

    std::vector<float> qa((size_t)na), qwh((size_t)nw);
    cuda_check(cudaMemcpy(qa.data(), dqa.p, na * sizeof(float), cudaMemcpyDeviceToHost), "D2H qa");
    cuda_check(cudaMemcpy(qwh.data(), qw, nw * sizeof(float), cudaMemcpyDeviceToHost), "D2H qw");

    // resolved scales snapshot (exec.hpp:248-259), host qfb (glibc, bitwise)
    const std::vector<double> sw = qfb::resolve_scale(std::span<const double>(layer.scales.log_w_scale), layer.qcfg);
    std::vector<float> snap((size_t)c_out + 1);
    for (int64_t c = 0; c < c_out; ++c) snap[(size_t)c] = static_cast<float>(sw[(size_t)c]);
    snap[(size_t)c_out] = static_cast<float>(qfb::resolve_scale(
        layer.scales.log_a_scale, layer.qcfg, half_acts ? QFB_PREC_HALF : QFB_PREC_FULL));
    ectx.last_scales[layer_idx] = Tensor({c_out + 1}, std::move(snap), Precision::Full);

    if (ectx.plan.cache_weights && !use_cache) ectx.cached_weights[layer_idx] = Tensor(layer.weight.shape, qwh);
    const float* wq = use_cache ? ectx.cached_weights[layer_idx].data.data() : qwh.data();
    out = conv2d_raw(qa.data(), input.shape, wq, layer.weight.shape, layer.stride, layer.padding, ep);
  }
  if (!all_finite(out)) throw NonFiniteError("non-finite activations in layer " + layer.name);
  LayerTrace lt;
  lt.name = layer.name;
  ectx.trace.per_layer.push_back(std::move(lt));
  return out;
}

}  // namespace qf

// The qfb side of the device-view hooks: x, y, upstream, d_input and the
// scale vectors in device memory, the async qfb::DeviceView overloads on
// the context stream, one sync, results copied back.
qf::Tensor dropin_dv_fq(const qf::Tensor& x, std::span<const double> s, const qf::QuantConfig& cfg) {
  const int64_t C = x.shape[0], n = x.numel();
  std::vector<float> s32((size_t)C);
  qfb::check(qfb_cast_scales_f32(s.data(), C, s32.data()));
  DevBuf dx((size_t)n), dy((size_t)n), ds((size_t)C);
  cuda_check(cudaMemcpy(dx.p, x.data.data(), n * 4, cudaMemcpyHostToDevice), "H2D x");
  cuda_check(cudaMemcpy(ds.p, s32.data(), C * 4, cudaMemcpyHostToDevice), "H2D s");
  qfb::fake_quantize(ctx(), qfb::DeviceView{dx.p, QFB_F32, 1, C, n / C}, dy.p, ds.p, cfg.q_max());
  qfb::check(qfb_ctx_sync(ctx().get()));
  qf::Tensor y = x;
  cuda_check(cudaMemcpy(y.data.data(), dy.p, n * 4, cudaMemcpyDeviceToHost), "D2H y");
  return y;
}

qf::FakeQuantGrad dropin_dv_bwd(const qf::Tensor& x, std::span<const double> log_s, const qf::QuantConfig& cfg,
                                const qf::Tensor& up) {
  const int64_t C = x.shape[0], n = x.numel();
  const qfb_quant_config c = qfb::to_c(cfg);
  std::vector<double> fac((size_t)(2 * C));
  qfb::check(qfb_scale_grad_factors(log_s.data(), C, &c, QFB_PREC_FULL, fac.data(), fac.data() + C));
  DevBuf dx((size_t)n), du((size_t)n), dd((size_t)n), df((size_t)(4 * C)), dl((size_t)(2 * C));
  cuda_check(cudaMemcpy(dx.p, x.data.data(), n * 4, cudaMemcpyHostToDevice), "H2D x");
  cuda_check(cudaMemcpy(du.p, up.data.data(), n * 4, cudaMemcpyHostToDevice), "H2D up");
  double* f64 = reinterpret_cast<double*>(df.p);
  double* dls = reinterpret_cast<double*>(dl.p);
  cuda_check(cudaMemcpy(f64, fac.data(), 2 * C * 8, cudaMemcpyHostToDevice), "H2D factors");
  qfb::fake_quantize_backward(ctx(), qfb::DeviceView{dx.p, QFB_F32, 1, C, n / C}, du.p, dd.p, f64, f64 + C, dls,
                              false, cfg.q_max());
  qfb::check(qfb_ctx_sync(ctx().get()));
  qf::FakeQuantGrad g;
  g.d_input = qf::Tensor::zeros(x.shape);
  g.d_log_scale.resize((size_t)C);
  cuda_check(cudaMemcpy(g.d_input.data.data(), dd.p, n * 4, cudaMemcpyDeviceToHost), "D2H dx");
  cuda_check(cudaMemcpy(g.d_log_scale.data(), dls, C * 8, cudaMemcpyDeviceToHost), "D2H d_log_s");
  return g;
}

namespace qf {

// distill.hpp:125-141 on the GPU (qfb_distill_loss_host, bit-identical).
DistillLoss distill_loss(const Tensor& f_s, const Tensor& f_t, const Tensor& i_s, const Tensor& i_t,
                         double lambda_cos) {
  ++g_dropin_calls.distill_loss;
  auto l = translated([&] { return qfb::distill_loss(ctx(), f_s, f_t, i_s, i_t, lambda_cos); });
  DistillLoss r;
  r.total = l.total;
  r.mse_f = l.mse_f;
  r.mse_i = l.mse_i;
  r.cos_f = l.cos_f;
  r.cos_i = l.cos_i;
  r.d_features = std::move(l.d_features);
  r.d_descriptors = std::move(l.d_descriptors);
  return r;
}

}  // namespace qf
