// rf_* planner C-ABI of the product library (include/reforward_b200.h).
#include "reforward_b200.h"
#include "reforward_b200/planner.hpp"

#define RF_ABI_NAME "reforward_b200 1"
#include "capi_impl.inc"
