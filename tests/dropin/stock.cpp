// stock.cpp — the unmodified reference (namespace qf), built from its own
// headers under /root/reference with its Release flags. Test infrastructure.
#include <algorithm>
#include <cmath>

#include "quantfuse/distill.hpp"
#include "dropin.h"

#define DROPIN_FN dropin_run_stock
#include "dropin_cases.inc"

// the stock side of the device-view hooks: the reference's own calls
qf::Tensor dropin_dv_fq(const qf::Tensor& x, std::span<const double> s, const qf::QuantConfig& cfg) {
  return qf::fake_quantize(x, s, cfg);
}
qf::FakeQuantGrad dropin_dv_bwd(const qf::Tensor& x, std::span<const double> log_s, const qf::QuantConfig& cfg,
                                const qf::Tensor& up) {
  return qf::fake_quantize_backward(x, log_s, cfg, up);
}
