// Host-side re-forwarding planner: the C++ surface the training executor and
// the C-ABI are built on.  Names, argument meaning and error behaviour mirror
// the reference library's public interface (proj/include/reforward/*.hpp) so a
// caller of the reference compiles against this header unchanged; the
// implementation (paper_1808_00079_b200/csrc/planner/) is an independent
// restatement whose solutions must agree with the reference bit-for-bit
// (tests/test_planner_golden.py pins that against tests/golden/).
//
// Reference interface map (file:line in /root/reference/proj/include/reforward):
//   errors.hpp:8-37        Error hierarchy
//   bitset.hpp:11-103      VertexSet
//   graph.hpp:19-95        CompGraph (+Builder), interior_cost, normalize,
//                          reaches, is_linear_chain, structurally_equal
//   objective.hpp:14-74    Segment, Solution, objective_of, better_solution
//   lcg.hpp:13-188         Rational, analytic_uniform, AccessibilityGraph,
//                          build_accessibility_graph, shortest_stored_path, solve_lcg
//   closed_set.hpp:16-408  ClosedSet, classify, is_splitting_vertex, is_branched,
//                          enumerate_closed_sets, maximal_split, divide
//   division_tree.hpp:18-194 DivisionTreeNode, build_division_tree, dump, canonical_form
//   acg.hpp:19-600         build_max_term_list, solve_with_max_term, solve_acg
//   oracle.hpp:13-33       oracle_min
//   simulate.hpp:16-94     SimReport, simulate
//   policies.hpp:11-28     store_all, sqrt_heuristic_chain
//   generators.hpp:14-114  gen_chain, gen_residual, gen_inception, gen_dense, gen_random
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace reforward {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseError : Error { using Error::Error; };
struct ValidationError : Error { using Error::Error; };
struct SizeLimitError : Error { using Error::Error; };
struct DecompositionError : Error { using Error::Error; };
struct InternalError : Error { using Error::Error; };

using VertexId = std::uint32_t;
using Cost = std::int64_t;

// ---------------------------------------------------------------- VertexSet
// Runtime-sized bitset of vertex (or edge) indices.
class VertexSet {
 public:
  VertexSet() = default;
  explicit VertexSet(std::size_t n);
  VertexSet(const VertexSet& o) { copy_from(o); }
  VertexSet(VertexSet&& o) noexcept { move_from(std::move(o)); }
  VertexSet& operator=(const VertexSet& o) {
    if (this != &o) copy_from(o);
    return *this;
  }
  VertexSet& operator=(VertexSet&& o) noexcept {
    if (this != &o) move_from(std::move(o));
    return *this;
  }

  std::size_t capacity() const { return bits_; }
  bool test(std::size_t i) const { return (data()[i >> 6] >> (i & 63)) & 1u; }
  void set(std::size_t i) { data()[i >> 6] |= std::uint64_t{1} << (i & 63); }
  void reset(std::size_t i) { data()[i >> 6] &= ~(std::uint64_t{1} << (i & 63)); }
  void clear();

  std::size_t count() const;
  bool any() const;
  bool empty() const { return !any(); }

  VertexSet& operator|=(const VertexSet& o);
  VertexSet& operator&=(const VertexSet& o);
  bool operator==(const VertexSet& o) const;
  bool operator!=(const VertexSet& o) const { return !(*this == o); }
  bool is_subset_of(const VertexSet& o) const;
  bool intersects(const VertexSet& o) const;
  std::vector<std::uint32_t> to_indices() const;

  // Lexicographic order of the ascending index sequences; a proper prefix
  // sorts first.  Returns -1 / 0 / +1.
  static int compare_lex(const VertexSet& a, const VertexSet& b);

 private:
  // Sets of up to 512 vertices live inline: the planner's frontier scans copy
  // millions of them, and a heap allocation per copy dominated their cost.
  static constexpr std::size_t kInline = 8;
  std::size_t bits_ = 0;
  std::size_t nw_ = 0;
  std::uint64_t inl_[kInline] = {};
  std::unique_ptr<std::uint64_t[]> heap_;
  std::uint64_t* data() { return heap_ ? heap_.get() : inl_; }
  const std::uint64_t* data() const { return heap_ ? heap_.get() : inl_; }
  void copy_from(const VertexSet& o) {
    bits_ = o.bits_;
    nw_ = o.nw_;
    if (nw_ <= kInline) {
      heap_.reset();
      std::memcpy(inl_, o.data(), nw_ * sizeof(std::uint64_t));
    } else {
      heap_.reset(new std::uint64_t[nw_]);
      std::memcpy(heap_.get(), o.data(), nw_ * sizeof(std::uint64_t));
    }
  }
  void move_from(VertexSet&& o) {
    bits_ = o.bits_;
    nw_ = o.nw_;
    if (o.heap_) {
      heap_ = std::move(o.heap_);
    } else {
      heap_.reset();
      std::memcpy(inl_, o.inl_, nw_ * sizeof(std::uint64_t));
    }
    o.bits_ = o.nw_ = 0;
  }
};

// ---------------------------------------------------------------- CompGraph
class CompGraph {
 public:
  struct Builder {
    std::vector<std::string> names;
    std::vector<Cost> costs;
    std::vector<std::pair<VertexId, VertexId>> edges;
    bool strict = false;
    VertexId add_vertex(std::string name, Cost cost = 1);
    void add_edge(VertexId u, VertexId v) { edges.emplace_back(u, v); }
  };

  static CompGraph build(Builder b, std::vector<std::string>* warnings = nullptr);

  std::size_t n_vertices() const { return cost_.size(); }
  const std::vector<std::pair<VertexId, VertexId>>& edges() const { return edge_list_; }
  Cost cost(VertexId v) const { return cost_[v]; }
  const std::string& name(VertexId v) const { return label_[v]; }
  VertexId source() const { return src_; }
  VertexId sink() const { return dst_; }
  const std::vector<VertexId>& topo_order() const { return order_; }
  std::size_t topo_index(VertexId v) const { return rank_[v]; }
  const std::vector<VertexId>& successors(VertexId v) const { return succ_[v]; }
  const std::vector<VertexId>& predecessors(VertexId v) const { return pred_[v]; }
  bool has_edge(VertexId u, VertexId v) const { return fwd_[u].test(v); }
  bool connected(VertexId u, VertexId v) const { return nbr_[u].test(v); }
  bool reaches(VertexId u, VertexId v) const { return down_[u].test(v); }
  VertexSet interior() const;
  Cost interior_total() const;
  bool is_interior(VertexId v) const { return v != src_ && v != dst_; }
  std::optional<VertexId> find_vertex(const std::string& name) const;

  // Planner-internal bitset views: out-neighbours, undirected neighbours,
  // descendants (reflexive) and ancestors (reflexive).
  const VertexSet& out_set(VertexId v) const { return fwd_[v]; }
  const VertexSet& neighbour_set(VertexId v) const { return nbr_[v]; }
  const VertexSet& descendants(VertexId v) const { return down_[v]; }
  const VertexSet& ancestors(VertexId v) const { return up_[v]; }

 private:
  std::vector<std::string> label_;
  std::vector<Cost> cost_;
  std::vector<std::pair<VertexId, VertexId>> edge_list_;
  std::vector<std::vector<VertexId>> succ_, pred_;
  std::vector<VertexId> order_;
  std::vector<std::size_t> rank_;
  std::vector<VertexSet> fwd_, nbr_, down_, up_;
  VertexId src_ = 0, dst_ = 0;
};

Cost interior_cost(const CompGraph& g, const VertexSet& s);
CompGraph normalize(const CompGraph& g);
inline bool reaches(const CompGraph& g, VertexId u, VertexId v) { return g.reaches(u, v); }
bool is_linear_chain(const CompGraph& g);
bool structurally_equal(const CompGraph& a, const CompGraph& b);

// ---------------------------------------------------------------- objective
struct Segment {
  VertexSet members;
  Cost cost = 0;
};

struct Solution {
  VertexSet stored;
  Cost stored_cost = 0;
  Cost realized_max = 0;
  Cost total = 0;
  std::vector<Segment> segments;
  Cost candidate_max_term = 0;
};

Solution objective_of(const CompGraph& g, const VertexSet& stored);
bool better_solution(const Solution& a, const Solution& b);

// ---------------------------------------------------------------- LCG
struct Rational {
  std::int64_t num = 0;
  std::int64_t den = 1;
  static Rational make(std::int64_t n, std::int64_t d);
  bool operator==(const Rational& o) const { return num == o.num && den == o.den; }
  double value() const { return static_cast<double>(num) / static_cast<double>(den); }
};

struct AnalyticUniform {
  std::int64_t k = 0;
  Rational relative_cost;
};
AnalyticUniform analytic_uniform(std::int64_t n);

struct AccessibilityGraph {
  std::vector<VertexId> chain;
  Cost max_term = 0;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> edges;
  std::vector<Cost> prefix;
  Cost between(std::uint32_t i, std::uint32_t j) const { return prefix[j] - prefix[i + 1]; }
};

struct LcgSolution {
  VertexSet stored;
  Cost stored_cost = 0;
  Cost max_term = 0;
  Cost total = 0;
};

AccessibilityGraph build_accessibility_graph(const CompGraph& chain, Cost max_term);
LcgSolution shortest_stored_path(const CompGraph& chain, const AccessibilityGraph& ag);
LcgSolution solve_lcg(const CompGraph& chain);

// ---------------------------------------------------------------- closed sets
struct ClosedSet {
  VertexId entry = 0;
  VertexId exit = 0;
  VertexSet members;
  bool includes_direct_edge = false;
  Cost cost = 0;
  bool empty_interior() const { return !members.any(); }
};

enum class ClosedSetType { Splittable, Branched, NonBranched };
const char* to_string(ClosedSetType t);

ClosedSet make_closed_set(const CompGraph& g, VertexId entry, VertexId exit, VertexSet members,
                          bool includes_direct_edge);
ClosedSet whole_graph_set(const CompGraph& g);
bool is_splitting_vertex(const ClosedSet& cs, VertexId v, const CompGraph& g);
bool is_branched(const ClosedSet& cs, const CompGraph& g);
ClosedSetType classify(const ClosedSet& cs, const CompGraph& g);
std::vector<ClosedSet> enumerate_closed_sets(const CompGraph& g);
std::vector<ClosedSet> maximal_split(const ClosedSet& cs, const CompGraph& g);
std::vector<ClosedSet> divide(const ClosedSet& cs, const CompGraph& g);

// ---------------------------------------------------------------- division tree
struct DivisionTreeNode {
  enum class Kind { Set, Vertex };
  Kind kind = Kind::Set;
  ClosedSet set;
  VertexId vertex = 0;
  ClosedSetType type = ClosedSetType::NonBranched;
  bool divided = false;
  std::vector<std::unique_ptr<DivisionTreeNode>> children;
  std::uint32_t id = 0;

  bool is_vertex_leaf() const { return kind == Kind::Vertex; }
  bool is_leaf() const { return children.empty(); }
  Cost node_cost(const CompGraph& g) const { return kind == Kind::Vertex ? g.cost(vertex) : set.cost; }
};

std::unique_ptr<DivisionTreeNode> build_division_tree(const CompGraph& g);
std::size_t count_nodes(const DivisionTreeNode& node);
void dump_tree_text(const CompGraph& g, const DivisionTreeNode& node, std::string& out, int depth = 0);
std::string canonical_form(const CompGraph& g, const DivisionTreeNode& node);

// ---------------------------------------------------------------- ACG solver
std::vector<Cost> build_max_term_list(const CompGraph& g, const DivisionTreeNode& tree);

class AcgSolver;  // frontier engine, defined in the implementation
Solution solve_with_max_term(const CompGraph& g, const DivisionTreeNode& tree, Cost max_term,
                             AcgSolver* solver = nullptr);
Solution solve_acg(const CompGraph& g);

// ---------------------------------------------------------------- oracle / simulator / policies
Solution oracle_min(const CompGraph& g, std::size_t max_interior = 20);

struct SimReport {
  struct Event {
    std::string label;
    Cost live = 0;
  };
  std::vector<Event> timeline;
  Cost peak = 0;
  std::map<VertexId, std::uint32_t> recompute_count;
};
enum class BackwardOrder { ReverseTopoExit, ReverseTopoEntry };
SimReport simulate(const CompGraph& g, const Solution& sol,
                   BackwardOrder order = BackwardOrder::ReverseTopoExit);

Solution store_all(const CompGraph& g);
Solution sqrt_heuristic_chain(const CompGraph& g);

// ---------------------------------------------------------------- generators
CompGraph gen_chain(std::size_t n, const std::vector<Cost>& costs = {});
CompGraph gen_residual(std::size_t blocks, std::size_t len);
CompGraph gen_inception(std::size_t blocks, std::size_t width);
CompGraph gen_dense(std::size_t k);
CompGraph gen_random(std::size_t n, double p, std::uint64_t seed, Cost cost_min = 1, Cost cost_max = 1);

}  // namespace reforward
