// subst.cpp — the same reference headers, compiled with -Dqf=qfs (a
// separate copy of the reference, so both live in one binary) and with
// qfb substituted at the reference's own call sites, the INTEGRATION.md §2
// pattern:
//   frontend.hpp:112-113  fake_quantize(x, sa, cfg) / (weight, span, cfg)
//   frontend.hpp:221-229  fake_quantize_backward(weight, span, cfg, d_qw)
//                         fake_quantize_backward(x, log_a, cfg, d_qa, prec)
// by name (the two tokens are redirected to the qfb-backed overloads
// declared below; quant.hpp itself is included first and stays intact), and
//   exec.hpp:435-451      run_frontend's run_quant_conv calls
//   distill.hpp:236       train_scales' distill_loss call
// by symbol: this TU is built with -fno-inline, so those calls go through
// the symbols qfs::run_quant_conv / qfs::distill_loss, which subst_ops.cpp
// defines (strong definitions take precedence over the headers' inline
// copies at link time). Test infrastructure, not product code.
#include <algorithm>
#include <cmath>
#include <span>

#include "quantfuse/quant.hpp"
#include "quantfuse/tensor.hpp"

namespace qf {
Tensor qfb_fake_quantize(const Tensor& x, double s, const QuantConfig& cfg);
Tensor qfb_fake_quantize(const Tensor& x, std::span<const double> s, const QuantConfig& cfg);
FakeQuantGrad qfb_fake_quantize_backward(const Tensor& x, double log_s, const QuantConfig& cfg,
                                         const Tensor& upstream, Precision mode = Precision::Full);
FakeQuantGrad qfb_fake_quantize_backward(const Tensor& x, std::span<const double> log_s,
                                         const QuantConfig& cfg, const Tensor& upstream,
                                         Precision mode = Precision::Full);
}  // namespace qf

#define fake_quantize qfb_fake_quantize
#define fake_quantize_backward qfb_fake_quantize_backward
#include "quantfuse/distill.hpp"
#undef fake_quantize
#undef fake_quantize_backward

#include "dropin.h"

#define DROPIN_FN dropin_run_qfb
#include "dropin_cases.inc"
