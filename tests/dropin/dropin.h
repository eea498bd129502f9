// dropin.h — shared between the stock and the qfb-substituted translation
// units of the drop-in harness (test infrastructure, not product code).
// No reference types here: each TU sees its own copy of the reference
// (namespace qf, or qfs when compiled with -Dqf=qfs).
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

struct DropinSink {
  std::vector<std::pair<std::string, std::string>> blobs;
  void add(const std::string& name, const void* p, size_t n) {
    blobs.emplace_back(name, std::string(static_cast<const char*>(p), n));
  }
};

// How many times the substituted entry points ran (proves the reference's
// call sites were routed to qfb, not to the inline reference code).
struct DropinCalls {
  int64_t fake_quantize = 0;
  int64_t fake_quantize_backward = 0;
  int64_t run_quant_conv = 0;
  int64_t distill_loss = 0;
};
extern DropinCalls g_dropin_calls;

void dropin_run_stock(DropinSink& out);
void dropin_run_qfb(DropinSink& out);
