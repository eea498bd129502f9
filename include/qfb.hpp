// qfb.hpp — C++ mirror of the reference operator API (namespace qf,
// /root/reference/proj/include/quantfuse/quant.hpp) over the C-ABI qfb.h.
//
// Drop-in shape: the tensor-level overloads are templates over any tensor
// type with the reference's layout — `shape` (std::vector<int64_t>),
// `data` (std::vector<float>), `precision` (enum, 0 = Full, 1 =
// EmulatedHalf) — so code holding qf::Tensor switches from
//     qf::fake_quantize(x, s, cfg)                   (quant.hpp:136)
// to
//     qfb::fake_quantize(ctx, x, s, cfg)
// with the same result bits. Errors are thrown as the reference's
// exception types' mirrors (errors.hpp:11-33, exec.hpp:51); pass the
// reference's own types via QFB_ERROR_TYPES_FROM_QF to throw exactly those.
#pragma once

#include <cstdint>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "qfb.h"

namespace qfb {

// ------------------------------------------------------------ errors --
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValueError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NonFiniteError : std::runtime_error { using std::runtime_error::runtime_error; };
struct FusedPathError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(qfb_status st) {
  if (st == QFB_OK) return;
  const std::string msg = qfb_last_error();
  switch (st) {
    case QFB_ERR_SHAPE: throw ShapeError(msg);
    case QFB_ERR_VALUE: throw ValueError(msg);
    case QFB_ERR_IO: throw IoError(msg);
    case QFB_ERR_NONFINITE: throw NonFiniteError(msg);
    case QFB_ERR_FUSED_PATH: throw FusedPathError(msg);
    case QFB_ERR_CUDA: throw CudaError(msg);
    default: throw std::runtime_error(std::string(qfb_status_name(st)) + ": " + msg);
  }
}

// ------------------------------------------------------------ config --
enum class Precision : uint8_t { Full = 0, EmulatedHalf = 1 };  // tensor.hpp:23

// qf::QuantConfig (quant.hpp:35-61), same defaults.
struct QuantConfig {
  int bits = 8;
  double s_min = 1e-6;
  double s_min_half = 1e-4;
  double s_max = 64.0;
  double eps = 1e-8;

  int q_max() const { return (1 << (bits - 1)) - 1; }
  qfb_quant_config c() const { return {bits, 0, s_min, s_min_half, s_max, eps}; }
  void validate() const {
    const qfb_quant_config cc = c();
    check(qfb_quant_config_validate(&cc));
  }
};

template <class Cfg>
inline qfb_quant_config to_c(const Cfg& c) {
  return {c.bits, 0, c.s_min, c.s_min_half, c.s_max, c.eps};
}

template <class P>
inline qfb_precision to_prec(P p) {
  return static_cast<int>(p) == 1 ? QFB_PREC_HALF : QFB_PREC_FULL;
}

// ------------------------------------------------------- scale math --
inline double softplus(double x) { return qfb_softplus(x); }
inline double sigmoid(double x) { return qfb_sigmoid(x); }
inline double softplus_inv(double y) {
  double out = 0.0;
  check(qfb_softplus_inv(y, &out));
  return out;
}

template <class Cfg = QuantConfig>
inline double resolve_scale(double log_s, const Cfg& cfg = Cfg{},
                            qfb_precision prec = QFB_PREC_FULL) {
  const qfb_quant_config c = to_c(cfg);
  double s = 0.0;
  check(qfb_resolve_scales(&log_s, 1, &c, prec, &s));
  return s;
}

template <class Cfg = QuantConfig>
inline std::vector<double> resolve_scale(std::span<const double> log_s, const Cfg& cfg = Cfg{},
                                         qfb_precision prec = QFB_PREC_FULL) {
  const qfb_quant_config c = to_c(cfg);
  std::vector<double> s(log_s.size());
  check(qfb_resolve_scales(log_s.data(), (int64_t)log_s.size(), &c, prec, s.data()));
  return s;
}

// ------------------------------------------------------------ context --
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) { check(qfb_ctx_create(device, stream, &h_)); }
  ~Context() { qfb_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  qfb_ctx* get() const { return h_; }
  void sync() const { check(qfb_ctx_sync(h_)); }
  void set_stream(void* s) { check(qfb_ctx_set_stream(h_, s)); }

 private:
  qfb_ctx* h_ = nullptr;
};

// --------------------------------------------- host tensor (value) API --
namespace detail {
template <class T>
inline int64_t leading(const T& x) {
  if (x.shape.empty()) throw ShapeError("per-channel fake quantization of a rank-0 tensor");
  return x.shape[0];
}
}  // namespace detail

// qf::fake_quantize per-tensor (quant.hpp:136-146). Output tag == input tag.
template <class Tensor, class Cfg>
inline Tensor fake_quantize(Context& ctx, const Tensor& x, double s, const Cfg& cfg) {
  const qfb_quant_config c = to_c(cfg);
  Tensor out = x;
  const int64_t n = (int64_t)x.data.size();
  if (n == 0) return out;
  check(qfb_fake_quantize_host(ctx.get(), to_prec(x.precision), x.data.data(), out.data.data(), 1,
                               1, n, &s, &c));
  return out;
}

// qf::fake_quantize per-channel along axis 0 (quant.hpp:150-170).
template <class Tensor, class Cfg>
inline Tensor fake_quantize(Context& ctx, const Tensor& x, std::span<const double> s,
                            const Cfg& cfg) {
  const int64_t c0 = x.shape.empty() ? -1 : x.shape[0];
  if (c0 < 0 || (int64_t)s.size() != c0)
    throw ShapeError("fake_quantize: per-channel scale length " + std::to_string(s.size()) +
                     " != leading dim");
  const qfb_quant_config c = to_c(cfg);
  Tensor out = x;
  const int64_t n = (int64_t)x.data.size();
  check(qfb_fake_quantize_host(ctx.get(), to_prec(x.precision), x.data.data(), out.data.data(), 1,
                               c0, n / c0, s.data(), &c));
  return out;
}

// qf::int8_codes (quant.hpp:174-207); codes returned as int8 vector.
template <class Tensor, class Cfg>
inline std::vector<int8_t> int8_codes(Context& ctx, const Tensor& x, std::span<const double> s,
                                      const Cfg& cfg) {
  const qfb_quant_config c = to_c(cfg);
  const int64_t n = (int64_t)x.data.size();
  const int64_t ch = s.size() == 1 ? 1 : detail::leading(x);
  if ((int64_t)s.size() != ch) throw ShapeError("int8_codes: per-channel scale length mismatch");
  std::vector<int8_t> out((size_t)n);
  check(qfb_int8_codes_host(ctx.get(), x.data.data(), out.data(), 1, ch, n / ch, s.data(), &c));
  return out;
}

// qf::FakeQuantGrad (quant.hpp:209-212).
template <class Tensor>
struct FakeQuantGrad {
  Tensor d_input;
  std::vector<double> d_log_scale;
};

// qf::fake_quantize_backward per-tensor (quant.hpp:233-257).
template <class Tensor, class Cfg, class P>
inline FakeQuantGrad<Tensor> fake_quantize_backward(Context& ctx, const Tensor& x, double log_s,
                                                    const Cfg& cfg, const Tensor& upstream, P mode) {
  if (x.shape != upstream.shape) throw ShapeError("fake_quantize_backward: shape mismatch");
  const qfb_quant_config c = to_c(cfg);
  FakeQuantGrad<Tensor> g{upstream, {0.0}};
  g.d_input.precision = decltype(x.precision)(0);
  const int64_t n = (int64_t)x.data.size();
  check(qfb_fake_quantize_backward_host(ctx.get(), to_prec(mode), x.data.data(),
                                        upstream.data.data(), g.d_input.data.data(), 1, 1, n,
                                        &log_s, &c, g.d_log_scale.data(), 0));
  return g;
}

// qf::fake_quantize_backward per-channel (quant.hpp:261-294).
template <class Tensor, class Cfg, class P>
inline FakeQuantGrad<Tensor> fake_quantize_backward(Context& ctx, const Tensor& x,
                                                    std::span<const double> log_s,
                                                    const Cfg& cfg, const Tensor& upstream, P mode) {
  if (x.shape != upstream.shape) throw ShapeError("fake_quantize_backward: shape mismatch");
  const int64_t ch = detail::leading(x);
  if ((int64_t)log_s.size() != ch)
    throw ShapeError("fake_quantize_backward: per-channel scale length mismatch");
  const qfb_quant_config c = to_c(cfg);
  FakeQuantGrad<Tensor> g{upstream, std::vector<double>(log_s.size(), 0.0)};
  g.d_input.precision = decltype(x.precision)(0);
  const int64_t n = (int64_t)x.data.size();
  check(qfb_fake_quantize_backward_host(ctx.get(), to_prec(mode), x.data.data(),
                                        upstream.data.data(), g.d_input.data.data(), 1, ch,
                                        n / ch, log_s.data(), &c, g.d_log_scale.data(), 0));
  return g;
}

// ---------------------------------------------- device views (async) --
// [outer, channels, inner] view of a device buffer.
struct DeviceView {
  void* data;
  qfb_dtype dtype;
  int64_t outer, channels, inner;
};

inline void fake_quantize(Context& ctx, const DeviceView& x, void* y, const float* d_scale,
                          int q_max = 127, uint32_t flags = 0) {
  check(qfb_fq_fwd(ctx.get(), x.dtype, x.data, y, x.outer, x.channels, x.inner, d_scale, q_max,
                   flags));
}

inline void fake_quantize_backward(Context& ctx, const DeviceView& x, const void* up, void* dx,
                                   const double* d_scale64, const double* d_chain,
                                   double* d_log_s, bool accumulate = false, int q_max = 127) {
  check(qfb_fq_bwd(ctx.get(), x.dtype, x.data, up, dx, x.outer, x.channels, x.inner, d_scale64,
                   d_chain, q_max, d_log_s, accumulate ? 1 : 0));
}

// ------------------------------------------- QAT step pieces (f3) --
// qf::DistillLoss (distill.hpp:48-55) shape.
template <class Tensor>
struct DistillLoss {
  double total = 0.0, mse_f = 0.0, mse_i = 0.0, cos_f = 0.0, cos_i = 0.0;
  Tensor d_features;
  Tensor d_descriptors;
};

// qf::distill_loss (distill.hpp:126-141) on host tensors [C, ...]; computed
// on the GPU, bit-identical.
template <class Tensor>
inline DistillLoss<Tensor> distill_loss(Context& ctx, const Tensor& f_s, const Tensor& f_t, const Tensor& i_s,
                                        const Tensor& i_t, double lambda_cos) {
  if (f_s.shape != f_t.shape || i_s.shape != i_t.shape) throw ShapeError("distill_loss: student/teacher shape");
  if (f_s.shape.empty() || f_s.shape[0] < 1) throw ShapeError("distill_loss: channel dim must be >= 1");
  const int64_t fc = f_s.shape[0], ic = i_s.shape[0];
  DistillLoss<Tensor> out{0, 0, 0, 0, 0, f_s, i_s};
  out.d_features.precision = decltype(f_s.precision)(0);
  out.d_descriptors.precision = decltype(i_s.precision)(0);
  double o5[5];
  check(qfb_distill_loss_host(ctx.get(), f_s.data.data(), f_t.data.data(), fc, (int64_t)f_s.data.size() / fc,
                              i_s.data.data(), i_t.data.data(), ic, (int64_t)i_s.data.size() / ic, lambda_cos,
                              1.0, o5, out.d_features.data.data(), out.d_descriptors.data.data()));
  out.total = o5[0];
  out.mse_f = o5[1];
  out.mse_i = o5[2];
  out.cos_f = o5[3];
  out.cos_i = o5[4];
  return out;
}

// ------------------------------------------------------ formats (f4) --
// qf::load_tensor / save_tensor (tensor_io.hpp:115-125).
template <class Tensor>
inline Tensor load_tensor(const std::string& path) {
  qfb_tensor_file* t = nullptr;
  check(qfb_qsim_load(path.c_str(), &t));
  int32_t rank = 0, prec = 0;
  const int64_t* shape = nullptr;
  int64_t n = 0;
  const float* data = nullptr;
  check(qfb_qsim_info(t, &rank, &shape, &prec, &n, &data));
  Tensor out(std::vector<int64_t>(shape, shape + rank), std::vector<float>(data, data + n),
             static_cast<decltype(Tensor{}.precision)>(prec));
  qfb_qsim_free(t);
  return out;
}

template <class Tensor>
inline void save_tensor(const std::string& path, const Tensor& t) {
  check(qfb_qsim_save(path.c_str(), t.data.data(), (int32_t)t.shape.size(), t.shape.data(),
                      (int32_t)t.precision));
}

// qf::load_scales / save_scales (distill.hpp:320-362): name -> (log_w, log_a).
using ScaleMap = std::map<std::string, std::pair<std::vector<double>, double>>;

inline ScaleMap load_scales(const std::string& path) {
  qfb_scales* sc = nullptr;
  check(qfb_qscl_load(path.c_str(), &sc));
  ScaleMap out;
  for (int32_t i = 0; i < qfb_qscl_count(sc); ++i) {
    const char* name = nullptr;
    const double* w = nullptr;
    int64_t cnt = 0;
    double a = 0.0;
    check(qfb_qscl_layer(sc, i, &name, &w, &cnt, &a));
    out[name] = {std::vector<double>(w, w + cnt), a};
  }
  qfb_qscl_free(sc);
  return out;
}

// Any qf::ScaleSet-shaped value (by_layer: name -> {log_w_scale, log_a_scale}).
template <class SetT>
inline void save_scales(const std::string& path, const SetT& set) {
  std::vector<const char*> names;
  std::vector<const double*> w;
  std::vector<int64_t> counts;
  std::vector<double> a;
  for (const auto& [name, p] : set.by_layer) {
    names.push_back(name.c_str());
    w.push_back(p.log_w_scale.data());
    counts.push_back((int64_t)p.log_w_scale.size());
    a.push_back(p.log_a_scale);
  }
  check(qfb_qscl_save(path.c_str(), (int32_t)names.size(), names.data(), w.data(), counts.data(), a.data()));
}

}  // namespace qfb
