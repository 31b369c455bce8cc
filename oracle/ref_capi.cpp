// TEST INFRASTRUCTURE — parity oracle, never linked into the product.
//
// Compiles the reference planner itself (header-only C++20 under
// /root/reference/proj/include/reforward, read in place, never copied) behind
// the same rf_* C-ABI the product exports, so tests can call both libraries
// with identical arguments.  io.hpp is skipped (it needs the un-vendored
// nlohmann/json); nothing on the planner path uses it.
//
// Built by oracle/Makefile into oracle/_ref/libreforward_ref.so.
#include "reforward/acg.hpp"
#include "reforward/closed_set.hpp"
#include "reforward/division_tree.hpp"
#include "reforward/generators.hpp"
#include "reforward/graph.hpp"
#include "reforward/lcg.hpp"
#include "reforward/objective.hpp"
#include "reforward/oracle.hpp"
#include "reforward/policies.hpp"
#include "reforward/simulate.hpp"

#include "reforward_b200.h"

#define RF_ABI_NAME "reforward_ref 1"
#include "../paper_1808_00079_b200/csrc/planner/capi_impl.inc"
