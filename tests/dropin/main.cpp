// main.cpp — drop-in harness driver: runs the reference workload twice,
// once through the unmodified reference and once with qfb at the
// reference's call sites, and compares every result byte for byte.
// Prints one JSON line; exit status 0 iff every blob is identical and every
// substituted entry point was reached. Test infrastructure.
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>

#include "dropin.h"

int main() {
  DropinSink stock, sub;
  try {
    dropin_run_stock(stock);
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"stage\": \"stock\", \"error\": \"%s\"}\n", e.what());
    return 2;
  }
  try {
    dropin_run_qfb(sub);
  } catch (const std::exception& e) {
    std::printf("{\"ok\": false, \"stage\": \"qfb\", \"error\": \"%s\"}\n", e.what());
    return 3;
  }
  size_t bytes = 0, mismatched = 0, device_view = 0;
  std::string first_bad;
  const bool same_count = stock.blobs.size() == sub.blobs.size();
  for (size_t i = 0; same_count && i < stock.blobs.size(); ++i) {
    const auto& a = stock.blobs[i];
    const auto& b = sub.blobs[i];
    bytes += a.second.size();
    if (a.first.rfind("device_view", 0) == 0) ++device_view;
    if (a.first != b.first || a.second != b.second) {
      if (first_bad.empty()) first_bad = a.first;
      ++mismatched;
    }
  }
  const DropinCalls& c = g_dropin_calls;
  const bool routed = c.fake_quantize > 0 && c.fake_quantize_backward > 0 && c.run_quant_conv > 0 && c.distill_loss > 0;
  const bool ok = same_count && mismatched == 0 && routed;
  std::printf(
      "{\"ok\": %s, \"blobs\": %zu, \"bytes\": %zu, \"mismatched\": %zu, \"device_view_blobs\": %zu, "
      "\"first_mismatch\": \"%s\", "
      "\"calls\": {\"fake_quantize\": %lld, \"fake_quantize_backward\": %lld, \"run_quant_conv\": %lld, "
      "\"distill_loss\": %lld}}\n",
      ok ? "true" : "false", stock.blobs.size(), bytes, mismatched, device_view, first_bad.c_str(), (long long)c.fake_quantize,
      (long long)c.fake_quantize_backward, (long long)c.run_quant_conv, (long long)c.distill_loss);
  return ok ? 0 : 1;
}
