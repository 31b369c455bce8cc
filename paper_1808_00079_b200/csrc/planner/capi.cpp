// rf_* planner C-ABI of the product library (include/reforward_b200.h).
#include "reforward_b200.h"
#include "reforward_b200/planner.hpp"

#define RF_ABI_NAME "reforward_b200 1"
#include "capi_impl.inc"

namespace rfexec {
// Shared with the executor / kernel entry points so rf_last_error() reports
// their failures too.
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace rfexec
