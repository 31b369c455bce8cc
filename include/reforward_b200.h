/* C-ABI of the B200 re-forwarding framework (libreforward_b200.so).
 *
 * Plain pointers, sizes and opaque handles only; no torch or C++ types cross
 * this boundary.  Two groups of entry points:
 *
 *  1. rf_*   — the host planner.  Each call stands in for the reference C++
 *              interface named beside it (file:line under
 *              /root/reference/proj/include/reforward/); a ctypes / cgo / JNI
 *              binding of the reference would bind exactly these.  The same
 *              ABI is compiled against the reference headers into
 *              oracle/_ref/libreforward_ref.so, which is how parity is checked.
 *  2. rfx_*  — the re-forward training executor and its sm_100a kernels (no
 *              reference counterpart: the reference stops at the plan; these
 *              are the "train step" the plan drives).
 *
 * Error convention: every int-returning call returns RF_OK (0) or one of the
 * RF_E_* codes; rf_last_error() returns the message of the last failure on the
 * calling thread.  Reference exception -> code: ParseError 1, ValidationError
 * 2, SizeLimitError 3, DecompositionError 4, InternalError 5 (errors.hpp:8-37).
 */
#ifndef REFORWARD_B200_H_
#define REFORWARD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RF_OK 0
#define RF_E_PARSE 1
#define RF_E_VALIDATION 2
#define RF_E_SIZE_LIMIT 3
#define RF_E_DECOMPOSITION 4
#define RF_E_INTERNAL 5
#define RF_E_ARGUMENT 6
#define RF_E_CUDA 7
#define RF_E_UNKNOWN 9

/* Last error message on this thread ("" if none). */
const char* rf_last_error(void);
/* ABI version string, e.g. "reforward_b200 1" or "reforward_ref 1". */
const char* rf_abi_name(void);

/* ------------------------------------------------------------ graph-core */
typedef struct rf_graph rf_graph; /* an immutable, normalized CompGraph */

/* CompGraph::Builder + CompGraph::build (graph.hpp:23-51, 140-241).
 * names: n C strings; costs: n; edges: 2*n_edges vertex indices (u0,v0,u1,v1..).
 * warnings (optional): newline-separated lenient-mode warnings. */
int rf_graph_build(int32_t n, const char* const* names, const int64_t* costs, int32_t n_edges,
                   const uint32_t* edges, int32_t strict, rf_graph** out, char* warnings,
                   size_t warnings_cap);
void rf_graph_free(rf_graph* g);
int32_t rf_graph_num_vertices(const rf_graph* g);              /* graph.hpp:55 */
int32_t rf_graph_num_edges(const rf_graph* g);                 /* graph.hpp:56 */
int rf_graph_edges(const rf_graph* g, uint32_t* out_pairs);    /* sorted (u,v) pairs */
int64_t rf_graph_cost(const rf_graph* g, uint32_t v);          /* graph.hpp:57 */
const char* rf_graph_name(const rf_graph* g, uint32_t v);      /* graph.hpp:58 */
uint32_t rf_graph_source(const rf_graph* g);                   /* graph.hpp:59 */
uint32_t rf_graph_sink(const rf_graph* g);                     /* graph.hpp:60 */
int rf_graph_topo_order(const rf_graph* g, uint32_t* out);     /* graph.hpp:62 */
int32_t rf_graph_reaches(const rf_graph* g, uint32_t u, uint32_t v); /* graph.hpp:254 */
int32_t rf_graph_is_linear_chain(const rf_graph* g);           /* graph.hpp:258 */
int64_t rf_graph_interior_total(const rf_graph* g);            /* graph.hpp:85 */
int rf_graph_normalize(const rf_graph* g, rf_graph** out);     /* graph.hpp:244 */

/* ------------------------------------------------------------ solutions
 * A solution is returned as a stored mask (uint8 per vertex id) plus scalars;
 * segment_of (optional, n entries) receives the segment index of every
 * non-stored interior vertex and -1 elsewhere (objective.hpp:14-28). */
typedef struct rf_solution_info {
  int64_t stored_cost;
  int64_t realized_max;
  int64_t total;
  int64_t candidate_max_term;
  int32_t n_stored;
  int32_t n_segments;
} rf_solution_info;

int rf_objective_of(const rf_graph* g, const uint8_t* stored_mask, rf_solution_info* info,
                    int32_t* segment_of);                                  /* objective.hpp:33 */
int rf_solve_acg(const rf_graph* g, uint8_t* stored_mask, rf_solution_info* info,
                 int32_t* segment_of);                                     /* acg.hpp:579 */
int rf_solve_with_max_term(const rf_graph* g, int64_t max_term, uint8_t* stored_mask,
                           rf_solution_info* info, int32_t* segment_of);   /* acg.hpp:555 */
int rf_solve_lcg(const rf_graph* g, uint8_t* stored_mask, int64_t* stored_cost,
                 int64_t* max_term, int64_t* total);                       /* lcg.hpp:158 */
int rf_oracle_min(const rf_graph* g, int32_t max_interior, uint8_t* stored_mask,
                  rf_solution_info* info, int32_t* segment_of);            /* oracle.hpp:13 */
int rf_store_all(const rf_graph* g, uint8_t* stored_mask, rf_solution_info* info); /* policies.hpp:12 */
int rf_sqrt_heuristic_chain(const rf_graph* g, uint8_t* stored_mask, rf_solution_info* info); /* policies.hpp:17 */
int rf_analytic_uniform(int64_t n, int64_t* k, int64_t* num, int64_t* den); /* lcg.hpp:36 */

/* simulate (simulate.hpp:38): order 0 = ReverseTopoExit, 1 = ReverseTopoEntry.
 * recompute (optional, n entries): times each vertex is re-forwarded. */
int rf_simulate(const rf_graph* g, const uint8_t* stored_mask, int32_t order, int64_t* peak,
                int32_t* n_events, uint32_t* recompute);

/* ------------------------------------------------------------ closed sets / tree
 * Text dumps use one line per set: "entry exit direct cost m1,m2,..\n" with
 * vertex ids; the tree dump is dump_tree_text's format. `needed` receives the
 * full length (+1 for NUL); the call fails with RF_E_ARGUMENT if cap is short. */
int rf_enumerate_closed_sets(const rf_graph* g, char* buf, size_t cap, size_t* needed); /* closed_set.hpp:193 */
int rf_divide_whole(const rf_graph* g, int32_t* type, char* buf, size_t cap, size_t* needed); /* closed_set.hpp:361 */
int rf_maximal_split_whole(const rf_graph* g, char* buf, size_t cap, size_t* needed); /* closed_set.hpp:271 */
int rf_division_tree_text(const rf_graph* g, char* buf, size_t cap, size_t* needed); /* division_tree.hpp:162 */
int rf_division_tree_canonical(const rf_graph* g, char* buf, size_t cap, size_t* needed); /* division_tree.hpp:183 */
int rf_division_tree_count(const rf_graph* g, int64_t* nodes);                      /* division_tree.hpp:155 */
int rf_max_term_list(const rf_graph* g, int64_t* out, int32_t cap, int32_t* n_out); /* acg.hpp:19 */

/* ------------------------------------------------------------ generators (generators.hpp) */
int rf_gen_chain(int32_t n, const int64_t* costs, int32_t n_costs, rf_graph** out);
int rf_gen_residual(int32_t blocks, int32_t len, rf_graph** out);
int rf_gen_inception(int32_t blocks, int32_t width, rf_graph** out);
int rf_gen_dense(int32_t k, rf_graph** out);
int rf_gen_random(int32_t n, double p, uint64_t seed, int64_t cost_min, int64_t cost_max,
                  rf_graph** out);

#ifdef __cplusplus
}
#endif

#include "reforward_b200_exec.h"

#endif /* REFORWARD_B200_H_ */
