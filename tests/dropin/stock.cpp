// stock.cpp — the unmodified reference (namespace qf), built from its own
// headers under /root/reference with its Release flags. Test infrastructure.
#include <algorithm>
#include <cmath>

#include "quantfuse/distill.hpp"
#include "dropin.h"

#define DROPIN_FN dropin_run_stock
#include "dropin_cases.inc"
