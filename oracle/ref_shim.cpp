// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY. Compiled by oracle/Makefile directly
// from /root/reference/proj/include (nothing copied into this repo) into
// oracle/_ref/libqfref.so. Used (a) to pin the C restatement in
// oracle/qf_oracle.c bitwise against the reference itself, (b) to generate
// tests/golden/ fixtures, and (c) as the reference CPU arm of bench.py
// (`cpu_baseline.kind == "reference"`). The product never loads it.
//
// Built with the reference's own Release flags (-std=c++20 -O3 -DNDEBUG,
// proj/CMakeLists.txt:2-8), no -march, like its CMake build.

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <span>
#include <thread>
#include <vector>

#include "quantfuse/distill.hpp"
#include "quantfuse/exec.hpp"
#include "quantfuse/half.hpp"
#include "quantfuse/quant.hpp"
#include "quantfuse/rng.hpp"
#include "quantfuse/tensor.hpp"
#include "quantfuse/tensor_io.hpp"

namespace {

qf::QuantConfig to_cfg(const int32_t bits, const double* d4) {
  qf::QuantConfig c;
  c.bits = bits;
  c.s_min = d4[0];
  c.s_min_half = d4[1];
  c.s_max = d4[2];
  c.eps = d4[3];
  return c;
}

qf::Precision prec_of(int half) {
  return half ? qf::Precision::EmulatedHalf : qf::Precision::Full;
}

// Error codes mirror include/qfb.h.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const qf::ShapeError&) {
    return 1;
  } catch (const qf::ValueError&) {
    return 2;
  } catch (const qf::IoError&) {
    return 3;
  } catch (const qf::NonFiniteError&) {
    return 4;
  } catch (const qf::FusedPathError&) {
    return 6;
  } catch (...) {
    return 99;
  }
}

}  // namespace

extern "C" {

// cfg passed as bits + {s_min, s_min_half, s_max, eps}.
int ref_cfg_validate(int32_t bits, const double* d4) {
  return guarded([&] { to_cfg(bits, d4).validate(); });
}

double ref_softplus(double x) { return qf::softplus(x); }
double ref_sigmoid(double x) { return qf::sigmoid(x); }
int ref_softplus_inv(double y, double* out) {
  return guarded([&] { *out = qf::softplus_inv(y); });
}
int ref_resolve_scale(double log_s, int32_t bits, const double* d4, int half,
                      double* out) {
  return guarded([&] { *out = qf::resolve_scale(log_s, to_cfg(bits, d4), prec_of(half)); });
}

float ref_fq_value(float x, float s, float q) { return qf::fake_quantize_value(x, s, q); }
uint16_t ref_f32_to_f16_bits(float v) { return qf::f32_to_f16_rne(v); }
float ref_f16_bits_to_f32(uint16_t h) { return qf::f16_to_f32(h); }
float ref_round_to_half(float v, int* sat) {
  bool b = false;
  const float r = qf::round_to_half(v, &b);
  if (sat) *sat = b ? 1 : 0;
  return r;
}
double ref_pairwise_sum(const double* p, int64_t n) { return qf::pairwise_sum(p, n); }

// qf::fake_quantize on a tensor of `shape` (rank<=4). nscale == 1 ->
// per-tensor overload (quant.hpp:136), else per-channel (quant.hpp:150).
int ref_fake_quantize(const float* x, const int64_t* shape, int rank, int half,
                      const double* s, int64_t nscale, int32_t bits,
                      const double* d4, float* y) {
  return guarded([&] {
    std::vector<int64_t> sh(shape, shape + rank);
    const int64_t n = qf::Tensor::numel_of(sh);
    qf::Tensor t(sh, std::vector<float>(x, x + n), prec_of(half));
    const qf::QuantConfig cfg = to_cfg(bits, d4);
    qf::Tensor out = nscale == 1
                         ? qf::fake_quantize(t, s[0], cfg)
                         : qf::fake_quantize(t, std::span<const double>(s, nscale), cfg);
    std::memcpy(y, out.data.data(), sizeof(float) * n);
  });
}

// Same, forcing the per-channel overload even for one channel.
int ref_fake_quantize_pc(const float* x, const int64_t* shape, int rank, int half,
                         const double* s, int64_t nscale, int32_t bits,
                         const double* d4, float* y) {
  return guarded([&] {
    std::vector<int64_t> sh(shape, shape + rank);
    const int64_t n = qf::Tensor::numel_of(sh);
    qf::Tensor t(sh, std::vector<float>(x, x + n), prec_of(half));
    qf::Tensor out = qf::fake_quantize(t, std::span<const double>(s, nscale), to_cfg(bits, d4));
    std::memcpy(y, out.data.data(), sizeof(float) * n);
  });
}

int ref_int8_codes(const float* x, const int64_t* shape, int rank,
                   const double* s, int64_t nscale, int per_channel,
                   int32_t bits, const double* d4, int8_t* codes) {
  return guarded([&] {
    std::vector<int64_t> sh(shape, shape + rank);
    const int64_t n = qf::Tensor::numel_of(sh);
    qf::Tensor t(sh, std::vector<float>(x, x + n));
    const qf::QuantConfig cfg = to_cfg(bits, d4);
    qf::IntTensor out = per_channel ? qf::int8_codes(t, std::span<const double>(s, nscale), cfg)
                                    : qf::int8_codes(t, s[0], cfg);
    std::memcpy(codes, out.data.data(), static_cast<size_t>(n));
  });
}

// qf::fake_quantize_backward; per_channel selects the span overload.
int ref_fq_backward(const float* x, const float* up, const int64_t* shape,
                    int rank, const double* log_s, int64_t nscale,
                    int per_channel, int half, int32_t bits, const double* d4,
                    float* dx, double* d_log_s) {
  return guarded([&] {
    std::vector<int64_t> sh(shape, shape + rank);
    const int64_t n = qf::Tensor::numel_of(sh);
    qf::Tensor tx(sh, std::vector<float>(x, x + n), prec_of(half));
    qf::Tensor tu(sh, std::vector<float>(up, up + n));
    const qf::QuantConfig cfg = to_cfg(bits, d4);
    qf::FakeQuantGrad g =
        per_channel ? qf::fake_quantize_backward(tx, std::span<const double>(log_s, nscale),
                                                 cfg, tu, prec_of(half))
                    : qf::fake_quantize_backward(tx, log_s[0], cfg, tu, prec_of(half));
    if (dx) std::memcpy(dx, g.d_input.data.data(), sizeof(float) * n);
    for (size_t i = 0; i < g.d_log_scale.size(); ++i) d_log_s[i] = g.d_log_scale[i];
  });
}

// qf::demote_half on a flat tensor; returns overflow count via *ovf.
int ref_demote_half(const float* x, int64_t n, float* y, uint64_t* ovf) {
  return guarded([&] {
    qf::Tensor t({n}, std::vector<float>(x, x + n));
    qf::Tensor d = qf::demote_half(t);
    std::memcpy(y, d.data.data(), sizeof(float) * n);
    if (ovf) *ovf = d.half_overflows;
  });
}

// relu(add(a, b)) then optional demote (exec.hpp:438,443,447).
int ref_residual_join(const float* a, const float* b, int64_t n, int half, float* y) {
  return guarded([&] {
    qf::Tensor ta({n}, std::vector<float>(a, a + n));
    qf::Tensor tb({n}, std::vector<float>(b, b + n));
    qf::Tensor r = qf::relu(qf::add(ta, tb));
    if (half) r = qf::demote_half(r);
    std::memcpy(y, r.data.data(), sizeof(float) * n);
  });
}

uint64_t ref_rng_word(uint64_t seed, uint64_t stream, uint64_t i) {
  return qf::CounterRng{seed, stream}.word(i);
}
double ref_rng_uniform(uint64_t seed, uint64_t stream, uint64_t i) {
  return qf::CounterRng{seed, stream}.uniform(i);
}
double ref_rng_normal(uint64_t seed, uint64_t stream, uint64_t i) {
  return qf::CounterRng{seed, stream}.normal(i);
}

// ---------------------------------------------------------------------
// Reference CPU arm for bench.py: the per-channel activation FQ forward
// (quant.hpp:150) and scale-only backward (quant.hpp:261) over a table of
// quant points, each a [C, H*W] tensor with its own log scales. Work items
// (quant points) are distributed over `threads` host threads (the reference
// functions are pure and reentrant); threads <= 1 runs inline.
// Tensors are constructed before the clock starts; only the reference
// calls are timed. Returns wall seconds in *seconds.
// ---------------------------------------------------------------------
int ref_bench_points(int32_t npoints, const float* const* x,
                     const float* const* up, const int64_t* channels,
                     const int64_t* inner, const double* const* log_s,
                     int half, int do_fwd, int do_bwd, int32_t threads,
                     int32_t reps, double* seconds, double* checksum) {
  return guarded([&] {
    const qf::QuantConfig cfg;
    std::vector<qf::Tensor> tx, tu;
    std::vector<std::vector<double>> sv;
    for (int32_t p = 0; p < npoints; ++p) {
      const int64_t n = channels[p] * inner[p];
      tx.emplace_back(std::vector<int64_t>{channels[p], inner[p]},
                      std::vector<float>(x[p], x[p] + n), prec_of(half));
      tu.emplace_back(std::vector<int64_t>{channels[p], inner[p]},
                      std::vector<float>(up[p], up[p] + n));
      std::vector<double> ls(log_s[p], log_s[p] + channels[p]);
      sv.push_back(qf::resolve_scale(std::span<const double>(ls), cfg, prec_of(half)));
    }
    std::vector<double> sums(static_cast<size_t>(npoints), 0.0);
    auto work = [&](int32_t p) {
      double acc = 0.0;
      if (do_fwd) {
        qf::Tensor y = qf::fake_quantize(tx[p], std::span<const double>(sv[p]), cfg);
        acc += y.data[0];
      }
      if (do_bwd) {
        qf::FakeQuantGrad g = qf::fake_quantize_backward(
            tx[p], std::span<const double>(log_s[p], channels[p]), cfg, tu[p], prec_of(half));
        acc += g.d_log_scale[0];
      }
      sums[static_cast<size_t>(p)] += acc;
    };
    const auto t0 = std::chrono::steady_clock::now();
    for (int32_t r = 0; r < reps; ++r) {
      if (threads <= 1) {
        for (int32_t p = 0; p < npoints; ++p) work(p);
      } else {
        std::atomic<int32_t> next{0};
        std::vector<std::thread> pool;
        for (int32_t t = 0; t < threads; ++t) {
          pool.emplace_back([&] {
            for (int32_t p = next++; p < npoints; p = next++) work(p);
          });
        }
        for (auto& th : pool) th.join();
      }
    }
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    double cs = 0.0;
    for (double v : sums) cs += v;
    if (checksum) *checksum = cs;
  });
}

// ---------------------------------------------------------------------
// Reference CPU arm with the reference's OWN parallel schedule: per quant
// point the operator's scale pass (exec.hpp:248-259: resolve_scale per
// channel, cast to float), its fused quantization sweep through the
// engine's qf::Dispatcher (exec.hpp:127-146: `threads` workers, contiguous
// parts, sequential below 4096 elements; the sweep body is the per-channel
// form of exec.hpp:371-375, + round_to_half under HalfActivations as
// exec.hpp:365-367), then the trainer's backward call fake_quantize_backward
// (frontend.hpp:226-229), which the reference runs sequentially. threads =
// 0 is ExecutionPlan{threads = 0}. Output buffers are allocated before the
// clock starts, as the engine's arena would hold them.
// ---------------------------------------------------------------------
int ref_bench_sweeps(int32_t npoints, const float* const* x, const float* const* up,
                     const int64_t* channels, const int64_t* inner, const double* const* log_s,
                     int half, int do_bwd, int32_t threads, int32_t reps, double* seconds,
                     double* checksum) {
  return guarded([&] {
    const qf::QuantConfig cfg;
    const float q = static_cast<float>(cfg.q_max());
    std::vector<qf::Tensor> tx, tu;
    std::vector<std::vector<float>> qa;
    for (int32_t p = 0; p < npoints; ++p) {
      const int64_t n = channels[p] * inner[p];
      tx.emplace_back(std::vector<int64_t>{channels[p], inner[p]},
                      std::vector<float>(x[p], x[p] + n), prec_of(half));
      tu.emplace_back(std::vector<int64_t>{channels[p], inner[p]},
                      std::vector<float>(up[p], up[p] + n));
      qa.emplace_back(static_cast<size_t>(n));
    }
    qf::Dispatcher disp(threads);
    double cs = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int32_t r = 0; r < reps; ++r) {
      for (int32_t p = 0; p < npoints; ++p) {
        const int64_t C = channels[p], per = inner[p], n = C * per;
        std::vector<float> sw(static_cast<size_t>(C));
        for (int64_t c = 0; c < C; ++c)
          sw[static_cast<size_t>(c)] = static_cast<float>(qf::resolve_scale(log_s[p][c], cfg, prec_of(half)));
        const float* xi = tx[p].data.data();
        float* out = qa[p].data();
        disp.sweep(n, [&](int64_t lo, int64_t hi) {
          for (int64_t i = lo; i < hi; ++i) {
            float v = qf::fake_quantize_value(xi[i], sw[static_cast<size_t>(i / per)], q);
            if (half) v = qf::round_to_half(v);
            out[i] = v;
          }
        });
        cs += out[0];
        if (do_bwd) {
          qf::FakeQuantGrad g = qf::fake_quantize_backward(
              tx[p], std::span<const double>(log_s[p], static_cast<size_t>(C)), cfg, tu[p], prec_of(half));
          cs += g.d_log_scale[0];
        }
      }
    }
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (checksum) *checksum = cs;
  });
}

// ---------------------------------------------------------------------
// Formats (tensor_io.hpp, distill.hpp:287-362) and the distillation loss
// (distill.hpp:66-141), for the f3/f4 parity tests and golden fixtures.
// ---------------------------------------------------------------------
static int copy_out(const std::string& b, char* out, size_t cap, size_t* size) {
  *size = b.size();
  if (out) {
    if (cap < b.size()) return 2;
    std::memcpy(out, b.data(), b.size());
  }
  return 0;
}

int ref_serialize_tensor(const float* data, const int64_t* shape, int rank, int prec, char* out,
                         size_t cap, size_t* size) {
  int rc = 0;
  const int st = guarded([&] {
    std::vector<int64_t> sh(shape, shape + rank);
    int64_t n = 1;
    for (int64_t d : sh) n *= d;
    qf::Tensor t(sh, std::vector<float>(data, data + n), prec_of(prec));
    rc = copy_out(qf::serialize_tensor(t), out, cap, size);
  });
  return st ? st : rc;
}

// Parses one tensor at *offset; shape_out holds up to 8 dims, data_out up
// to cap_n floats (*numel is always set).
int ref_parse_tensor(const char* buf, size_t size, size_t* offset, int64_t* shape_out, int* rank,
                     int* prec, float* data_out, int64_t cap_n, int64_t* numel) {
  return guarded([&] {
    const std::string b(buf, size);
    size_t off = *offset;
    qf::Tensor t = qf::parse_tensor(b, off);
    *offset = off;
    *rank = (int)t.shape.size();
    for (size_t i = 0; i < t.shape.size() && i < 8; ++i) shape_out[i] = t.shape[i];
    *prec = (int)t.precision;
    *numel = (int64_t)t.data.size();
    if (data_out && (int64_t)t.data.size() <= cap_n)
      std::memcpy(data_out, t.data.data(), t.data.size() * 4);
  });
}

int ref_serialize_scales(int n, const char* const* names, const double* const* log_w,
                         const int64_t* counts, const double* log_a, char* out, size_t cap,
                         size_t* size) {
  int rc = 0;
  const int st = guarded([&] {
    qf::ScaleSet set;
    for (int i = 0; i < n; ++i) {
      qf::ScaleParams p;
      p.log_w_scale.assign(log_w[i], log_w[i] + counts[i]);
      p.log_a_scale = log_a[i];
      set.by_layer[names[i]] = p;
    }
    rc = copy_out(qf::serialize_scales(set), out, cap, size);
  });
  return st ? st : rc;
}

// parse_scales then serialize_scales (the reference's round trip).
int ref_scales_roundtrip(const char* buf, size_t size, char* out, size_t cap, size_t* osize) {
  int rc = 0;
  const int st = guarded([&] {
    const qf::ScaleSet set = qf::parse_scales(std::string(buf, size));
    rc = copy_out(qf::serialize_scales(set), out, cap, osize);
  });
  return st ? st : rc;
}

// Layer i (name order) of a parsed QSCL blob.
int ref_scales_layer(const char* buf, size_t size, int i, char* name, size_t name_cap,
                     double* log_w, int64_t cap_w, int64_t* count, double* log_a, int* n_layers) {
  return guarded([&] {
    const qf::ScaleSet set = qf::parse_scales(std::string(buf, size));
    *n_layers = (int)set.by_layer.size();
    int k = 0;
    for (const auto& [nm, p] : set.by_layer) {
      if (k++ != i) continue;
      std::snprintf(name, name_cap, "%s", nm.c_str());
      *count = (int64_t)p.log_w_scale.size();
      for (int64_t j = 0; j < *count && j < cap_w; ++j) log_w[j] = p.log_w_scale[(size_t)j];
      *log_a = p.log_a_scale;
    }
  });
}

// distill_loss over [C, H, W] feature/descriptor pairs (distill.hpp:126-141):
// out6 = {total, mse_f, mse_i, cos_f, cos_i, 0}; d_f / d_i gradients.
int ref_distill_loss(const float* fs, const float* ft, const int64_t* fshape, const float* is,
                     const float* it, const int64_t* ishape, double lambda, double* out6, float* d_f,
                     float* d_i) {
  return guarded([&] {
    auto mk = [](const float* p, const int64_t* sh) {
      std::vector<int64_t> v(sh, sh + 3);
      return qf::Tensor(v, std::vector<float>(p, p + v[0] * v[1] * v[2]));
    };
    const qf::DistillLoss dl = qf::distill_loss(mk(fs, fshape), mk(ft, fshape), mk(is, ishape),
                                                mk(it, ishape), lambda);
    out6[0] = dl.total;
    out6[1] = dl.mse_f;
    out6[2] = dl.mse_i;
    out6[3] = dl.cos_f;
    out6[4] = dl.cos_i;
    out6[5] = 0.0;
    std::memcpy(d_f, dl.d_features.data.data(), dl.d_features.data.size() * 4);
    std::memcpy(d_i, dl.d_descriptors.data.data(), dl.d_descriptors.data.size() * 4);
  });
}

}  // extern "C"
