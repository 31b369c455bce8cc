// Graph core, Eq. 1 scoring, exhaustive oracle, schedule simulator, baseline
// policies and topology generators.  Restates the behaviour of
// reference proj/include/reforward/{bitset,graph,objective,oracle,simulate,
// policies,generators}.hpp (see include/reforward_b200/planner.hpp for the map).
#include <algorithm>
#include <bit>
#include <cmath>
#include <queue>
#include <random>

#include "reforward_b200/planner.hpp"

namespace reforward {

// ============================================================ VertexSet
VertexSet::VertexSet(std::size_t n) : bits_(n), nw_((n + 63) / 64) {
  if (nw_ > kInline) heap_.reset(new std::uint64_t[nw_]());
}

void VertexSet::clear() { std::fill(data(), data() + nw_, 0); }

std::size_t VertexSet::count() const {
  std::size_t c = 0;
  const std::uint64_t* w = data();
  for (std::size_t i = 0; i < nw_; ++i) c += static_cast<std::size_t>(std::popcount(w[i]));
  return c;
}

bool VertexSet::any() const {
  const std::uint64_t* w = data();
  for (std::size_t i = 0; i < nw_; ++i)
    if (w[i]) return true;
  return false;
}

bool VertexSet::operator==(const VertexSet& o) const {
  return nw_ == o.nw_ && std::memcmp(data(), o.data(), nw_ * sizeof(std::uint64_t)) == 0;
}

VertexSet& VertexSet::operator|=(const VertexSet& o) {
  std::uint64_t* w = data();
  const std::uint64_t* v = o.data();
  for (std::size_t i = 0; i < nw_; ++i) w[i] |= v[i];
  return *this;
}

VertexSet& VertexSet::operator&=(const VertexSet& o) {
  std::uint64_t* w = data();
  const std::uint64_t* v = o.data();
  for (std::size_t i = 0; i < nw_; ++i) w[i] &= v[i];
  return *this;
}

bool VertexSet::is_subset_of(const VertexSet& o) const {
  const std::uint64_t *w = data(), *v = o.data();
  for (std::size_t i = 0; i < nw_; ++i)
    if (w[i] & ~v[i]) return false;
  return true;
}

bool VertexSet::intersects(const VertexSet& o) const {
  const std::uint64_t *w = data(), *v = o.data();
  for (std::size_t i = 0; i < nw_; ++i)
    if (w[i] & v[i]) return true;
  return false;
}

std::vector<std::uint32_t> VertexSet::to_indices() const {
  std::vector<std::uint32_t> idx;
  const std::uint64_t* w = data();
  for (std::size_t wi = 0; wi < nw_; ++wi)
    for (std::uint64_t x = w[wi]; x; x &= x - 1)
      idx.push_back(static_cast<std::uint32_t>(wi * 64 + static_cast<std::size_t>(std::countr_zero(x))));
  return idx;
}

int VertexSet::compare_lex(const VertexSet& a, const VertexSet& b) {
  // The first index present in exactly one set decides.  The set holding it
  // is smaller unless the other set has nothing at or past that index (then
  // the other set is a proper prefix and sorts first).
  const std::size_t nw = a.nw_;
  const std::uint64_t *aw = a.data(), *bw = b.data();
  for (std::size_t wi = 0; wi < nw; ++wi) {
    const std::uint64_t d = aw[wi] ^ bw[wi];
    if (d == 0) continue;
    const std::uint64_t bit = d & (~d + 1);
    const std::uint64_t* missing = (aw[wi] & bit) ? bw : aw;
    bool more = (missing[wi] & ~(bit - 1)) != 0;
    for (std::size_t k = wi + 1; !more && k < nw; ++k) more = missing[k] != 0;
    const bool a_has = (aw[wi] & bit) != 0;
    if (a_has) return more ? -1 : 1;
    return more ? 1 : -1;
  }
  return 0;
}

// ============================================================ CompGraph
VertexId CompGraph::Builder::add_vertex(std::string name, Cost cost) {
  names.push_back(std::move(name));
  costs.push_back(cost);
  return static_cast<VertexId>(names.size() - 1);
}

namespace {

// Lexicographically-smallest topological order (Kahn, smallest ready id
// first), as in reference graph.hpp:116-137.
std::vector<VertexId> smallest_first_toposort(const std::vector<std::vector<VertexId>>& succ,
                                              const std::vector<std::vector<VertexId>>& pred) {
  const std::size_t n = succ.size();
  std::vector<std::size_t> missing(n);
  std::priority_queue<VertexId, std::vector<VertexId>, std::greater<VertexId>> ready;
  for (VertexId v = 0; v < n; ++v) {
    missing[v] = pred[v].size();
    if (missing[v] == 0) ready.push(v);
  }
  std::vector<VertexId> order;
  order.reserve(n);
  while (!ready.empty()) {
    VertexId v = ready.top();
    ready.pop();
    order.push_back(v);
    for (VertexId w : succ[v])
      if (--missing[w] == 0) ready.push(w);
  }
  if (order.size() != n) throw ValidationError("graph contains a cycle");
  return order;
}

std::string unused_name(const std::vector<std::string>& taken, std::string name) {
  while (std::find(taken.begin(), taken.end(), name) != taken.end()) name.insert(0, "_");
  return name;
}

}  // namespace

CompGraph CompGraph::build(Builder b, std::vector<std::string>* warnings) {
  auto note = [warnings](const std::string& m) {
    if (warnings) warnings->push_back(m);
  };
  const std::size_t n_in = b.names.size();
  for (std::size_t i = 0; i < b.costs.size(); ++i)
    if (b.costs[i] < 0) throw ValidationError("negative cost on vertex '" + b.names[i] + "'");
  for (const auto& e : b.edges) {
    if (e.first >= n_in || e.second >= n_in) throw ValidationError("edge references unknown vertex");
    if (e.first == e.second) throw ValidationError("self-loop on vertex '" + b.names[e.first] + "'");
  }
  std::sort(b.edges.begin(), b.edges.end());
  if (auto it = std::adjacent_find(b.edges.begin(), b.edges.end()); it != b.edges.end()) {
    if (b.strict)
      throw ValidationError("duplicate edge " + b.names[it->first] + " -> " + b.names[it->second]);
    note("duplicate edges removed");
    b.edges.erase(std::unique(b.edges.begin(), b.edges.end()), b.edges.end());
  }

  // Vertices touched by no edge lie on no source-sink path (a lone vertex is
  // the exception: it is its own source and sink).
  if (n_in > 1) {
    std::vector<char> used(n_in, 0);
    for (const auto& e : b.edges) used[e.first] = used[e.second] = 1;
    if (std::find(used.begin(), used.end(), 0) != used.end()) {
      std::vector<VertexId> new_id(n_in, 0);
      Builder kept;
      kept.strict = b.strict;
      for (VertexId v = 0; v < n_in; ++v) {
        if (!used[v]) {
          if (b.strict) throw ValidationError("vertex '" + b.names[v] + "' lies on no source-sink path");
          note("pruned isolated vertex '" + b.names[v] + "'");
          continue;
        }
        new_id[v] = kept.add_vertex(b.names[v], b.costs[v]);
      }
      if (kept.names.empty()) throw ValidationError("graph has no connected vertices");
      for (const auto& e : b.edges) kept.add_edge(new_id[e.first], new_id[e.second]);
      b = std::move(kept);
    }
  }

  const std::size_t n0 = b.names.size();
  if (n0 == 0) throw ValidationError("graph has no vertices");

  std::vector<std::size_t> indeg(n0, 0), outdeg(n0, 0);
  for (const auto& e : b.edges) {
    ++outdeg[e.first];
    ++indeg[e.second];
  }

  CompGraph g;
  g.label_ = std::move(b.names);
  g.cost_ = std::move(b.costs);
  g.edge_list_ = std::move(b.edges);

  if (n0 == 1) {
    g.src_ = g.dst_ = 0;
  } else {
    std::vector<VertexId> roots, leaves;
    for (VertexId v = 0; v < n0; ++v) {
      if (indeg[v] == 0) roots.push_back(v);
      if (outdeg[v] == 0) leaves.push_back(v);
    }
    if (roots.size() == 1) {
      g.src_ = roots.front();
    } else {
      g.src_ = static_cast<VertexId>(g.label_.size());
      g.label_.push_back(unused_name(g.label_, "_s"));
      g.cost_.push_back(0);
      for (VertexId r : roots) g.edge_list_.emplace_back(g.src_, r);
    }
    if (leaves.size() == 1) {
      g.dst_ = leaves.front();
    } else {
      g.dst_ = static_cast<VertexId>(g.label_.size());
      g.label_.push_back(unused_name(g.label_, "_t"));
      g.cost_.push_back(0);
      for (VertexId l : leaves) g.edge_list_.emplace_back(l, g.dst_);
    }
  }

  const std::size_t n = g.label_.size();
  std::sort(g.edge_list_.begin(), g.edge_list_.end());
  g.succ_.assign(n, {});
  g.pred_.assign(n, {});
  g.fwd_.assign(n, VertexSet(n));
  g.nbr_.assign(n, VertexSet(n));
  for (const auto& [u, v] : g.edge_list_) {
    g.succ_[u].push_back(v);
    g.pred_[v].push_back(u);
    g.fwd_[u].set(v);
    g.nbr_[u].set(v);
    g.nbr_[v].set(u);
  }
  g.order_ = smallest_first_toposort(g.succ_, g.pred_);
  g.rank_.assign(n, 0);
  for (std::size_t i = 0; i < n; ++i) g.rank_[g.order_[i]] = i;

  g.down_.assign(n, VertexSet(n));
  for (std::size_t i = n; i-- > 0;) {
    const VertexId v = g.order_[i];
    g.down_[v].set(v);
    for (VertexId w : g.succ_[v]) g.down_[v] |= g.down_[w];
  }
  g.up_.assign(n, VertexSet(n));
  for (VertexId u = 0; u < n; ++u)
    for (auto w : g.down_[u].to_indices()) g.up_[w].set(u);
  return g;
}

VertexSet CompGraph::interior() const {
  VertexSet s(n_vertices());
  for (VertexId v = 0; v < n_vertices(); ++v)
    if (is_interior(v)) s.set(v);
  return s;
}

Cost CompGraph::interior_total() const {
  Cost t = 0;
  for (VertexId v = 0; v < n_vertices(); ++v)
    if (is_interior(v)) t += cost_[v];
  return t;
}

std::optional<VertexId> CompGraph::find_vertex(const std::string& name) const {
  for (VertexId v = 0; v < n_vertices(); ++v)
    if (label_[v] == name) return v;
  return std::nullopt;
}

Cost interior_cost(const CompGraph& g, const VertexSet& s) {
  Cost t = 0;
  for (auto v : s.to_indices()) t += g.cost(v);
  return t;
}

CompGraph normalize(const CompGraph& g) {
  CompGraph::Builder b;
  for (VertexId v = 0; v < g.n_vertices(); ++v) b.add_vertex(g.name(v), g.cost(v));
  for (const auto& e : g.edges()) b.add_edge(e.first, e.second);
  return CompGraph::build(std::move(b));
}

bool is_linear_chain(const CompGraph& g) {
  for (VertexId v = 0; v < g.n_vertices(); ++v)
    if (g.successors(v).size() > 1 || g.predecessors(v).size() > 1) return false;
  return true;
}

bool structurally_equal(const CompGraph& a, const CompGraph& b) {
  if (a.n_vertices() != b.n_vertices() || a.edges() != b.edges()) return false;
  if (a.source() != b.source() || a.sink() != b.sink()) return false;
  for (VertexId v = 0; v < a.n_vertices(); ++v)
    if (a.name(v) != b.name(v) || a.cost(v) != b.cost(v)) return false;
  return true;
}

// ============================================================ Eq. 1 scoring
// Segments are the weakly-connected components of the non-stored interior
// vertices (reference objective.hpp:33-65), listed by first topological
// appearance.  Components are discovered by flood fill in topo order.
Solution objective_of(const CompGraph& g, const VertexSet& stored) {
  const std::size_t n = g.n_vertices();
  Solution sol;
  sol.stored = stored;
  sol.stored_cost = interior_cost(g, stored);

  std::vector<char> open(n, 0), seen(n, 0);
  for (VertexId v = 0; v < n; ++v) open[v] = g.is_interior(v) && !stored.test(v);
  std::vector<VertexId> stack;
  for (VertexId root : g.topo_order()) {
    if (!open[root] || seen[root]) continue;
    Segment seg{VertexSet(n), 0};
    seen[root] = 1;
    stack.assign(1, root);
    while (!stack.empty()) {
      VertexId v = stack.back();
      stack.pop_back();
      seg.members.set(v);
      seg.cost += g.cost(v);
      for (const auto* adj : {&g.successors(v), &g.predecessors(v)})
        for (VertexId w : *adj)
          if (open[w] && !seen[w]) {
            seen[w] = 1;
            stack.push_back(w);
          }
    }
    sol.realized_max = std::max(sol.realized_max, seg.cost);
    sol.segments.push_back(std::move(seg));
  }
  sol.total = sol.stored_cost + sol.realized_max;
  sol.candidate_max_term = sol.realized_max;
  return sol;
}

bool better_solution(const Solution& a, const Solution& b) {
  if (a.total != b.total) return a.total < b.total;
  const auto na = a.stored.count(), nb = b.stored.count();
  if (na != nb) return na < nb;
  return VertexSet::compare_lex(a.stored, b.stored) < 0;
}

// ============================================================ oracle
Solution oracle_min(const CompGraph& g, std::size_t max_interior) {
  const auto inner = g.interior().to_indices();
  if (inner.size() > max_interior)
    throw SizeLimitError("oracle limited to " + std::to_string(max_interior) +
                         " interior vertices, graph has " + std::to_string(inner.size()));
  Solution best;
  bool have = false;
  const std::uint64_t subsets = std::uint64_t{1} << inner.size();
  for (std::uint64_t mask = 0; mask < subsets; ++mask) {
    VertexSet s(g.n_vertices());
    for (std::size_t i = 0; i < inner.size(); ++i)
      if ((mask >> i) & 1u) s.set(inner[i]);
    Solution cand = objective_of(g, s);
    if (!have || better_solution(cand, best)) {
      best = std::move(cand);
      have = true;
    }
  }
  return best;
}

// ============================================================ simulator
SimReport simulate(const CompGraph& g, const Solution& sol, BackwardOrder order) {
  SimReport rep;
  Cost live = 0;
  auto mark = [&](std::string what) {
    rep.peak = std::max(rep.peak, live);
    rep.timeline.push_back({std::move(what), live});
  };
  for (auto v : g.interior().to_indices()) rep.recompute_count[v] = 0;

  mark("forward start");
  for (VertexId v : g.topo_order()) {
    if (!g.is_interior(v)) continue;
    if (sol.stored.test(v)) {
      live += g.cost(v);
      mark("store " + g.name(v));
    } else {
      mark("compute " + g.name(v) + " (transient)");
    }
  }

  // One segment live at a time; visit by descending last (or first) position.
  const bool by_exit = order == BackwardOrder::ReverseTopoExit;
  std::vector<std::pair<std::size_t, std::size_t>> keyed;  // (key, segment)
  for (std::size_t s = 0; s < sol.segments.size(); ++s) {
    std::size_t key = by_exit ? 0 : g.n_vertices();
    for (auto v : sol.segments[s].members.to_indices())
      key = by_exit ? std::max(key, g.topo_index(v)) : std::min(key, g.topo_index(v));
    keyed.emplace_back(key, s);
  }
  std::sort(keyed.begin(), keyed.end(), [](const auto& x, const auto& y) { return x.first > y.first; });

  mark("backward start");
  for (const auto& ks : keyed) {
    const Segment& seg = sol.segments[ks.second];
    live += seg.cost;
    for (auto v : seg.members.to_indices()) ++rep.recompute_count[v];
    mark("re-forward segment " + std::to_string(ks.second));
    live -= seg.cost;
    mark("backward segment " + std::to_string(ks.second));
  }
  live -= sol.stored_cost;
  mark("backward done");
  if (rep.peak != sol.total)
    throw InternalError("simulated peak " + std::to_string(rep.peak) + " != solution total " +
                        std::to_string(sol.total));
  return rep;
}

// ============================================================ policies
Solution store_all(const CompGraph& g) { return objective_of(g, g.interior()); }

Solution sqrt_heuristic_chain(const CompGraph& g) {
  if (!is_linear_chain(g)) throw ValidationError("sqrt heuristic applies to linear chains only");
  const auto& ord = g.topo_order();
  const std::size_t n = ord.size() >= 2 ? ord.size() - 2 : 0;
  VertexSet s(g.n_vertices());
  if (n > 0) {
    std::size_t step = static_cast<std::size_t>(std::llround(std::sqrt(static_cast<double>(n))));
    step = std::max<std::size_t>(step, 1);
    for (std::size_t pos = step; pos < n; pos += step) s.set(ord[pos]);
  }
  return objective_of(g, s);
}

// ============================================================ generators
CompGraph gen_chain(std::size_t n, const std::vector<Cost>& costs) {
  if (n < 1) throw ValidationError("chain needs at least one interior vertex");
  CompGraph::Builder b;
  VertexId prev = b.add_vertex("s", 1);
  for (std::size_t i = 0; i < n; ++i) {
    VertexId v = b.add_vertex("v" + std::to_string(i + 1), i < costs.size() ? costs[i] : 1);
    b.add_edge(prev, v);
    prev = v;
  }
  b.add_edge(prev, b.add_vertex("t", 1));
  return CompGraph::build(std::move(b));
}

CompGraph gen_residual(std::size_t blocks, std::size_t len) {
  if (blocks < 1 || len < 1) throw ValidationError("residual needs blocks >= 1, len >= 1");
  CompGraph::Builder b;
  VertexId prev = b.add_vertex("s", 1);
  std::size_t next = 0;
  for (std::size_t k = 0; k < blocks; ++k) {
    const VertexId in = prev;
    for (std::size_t i = 0; i < len; ++i) {
      VertexId v = b.add_vertex("v" + std::to_string(++next), 1);
      b.add_edge(prev, v);
      prev = v;
    }
    if (len > 1) b.add_edge(in, prev);
  }
  b.add_edge(prev, b.add_vertex("t", 1));
  return CompGraph::build(std::move(b));
}

CompGraph gen_inception(std::size_t blocks, std::size_t width) {
  if (blocks < 1 || width < 1) throw ValidationError("inception needs blocks, width >= 1");
  CompGraph::Builder b;
  VertexId prev = b.add_vertex("s", 1);
  std::size_t next = 0;
  for (std::size_t k = 0; k < blocks; ++k) {
    VertexId join = b.add_vertex("j" + std::to_string(k + 1), 1);
    for (std::size_t w = 0; w < width; ++w) {
      VertexId p = b.add_vertex("p" + std::to_string(++next), 1);
      b.add_edge(prev, p);
      b.add_edge(p, join);
    }
    prev = join;
  }
  b.add_edge(prev, b.add_vertex("t", 1));
  return CompGraph::build(std::move(b));
}

CompGraph gen_dense(std::size_t k) {
  if (k < 1) throw ValidationError("dense needs at least one vertex");
  CompGraph::Builder b;
  VertexId s = b.add_vertex("s", 1);
  std::vector<VertexId> vs;
  for (std::size_t i = 0; i < k; ++i) vs.push_back(b.add_vertex("v" + std::to_string(i + 1), 1));
  VertexId t = b.add_vertex("t", 1);
  b.add_edge(s, vs.front());
  for (std::size_t i = 0; i < k; ++i)
    for (std::size_t j = i + 1; j < k; ++j) b.add_edge(vs[i], vs[j]);
  b.add_edge(vs.back(), t);
  return CompGraph::build(std::move(b));
}

CompGraph gen_random(std::size_t n, double p, std::uint64_t seed, Cost cost_min, Cost cost_max) {
  if (n < 1) throw ValidationError("random needs at least one vertex");
  if (p < 0.0 || p > 1.0) throw ValidationError("edge probability must be in [0, 1]");
  if (cost_min < 0 || cost_max < cost_min) throw ValidationError("bad cost range");
  // Same engine, distributions and draw order as the reference generator
  // (generators.hpp:93-114): n cost draws, then one coin per pair i<j.
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> coin(0.0, 1.0);
  std::uniform_int_distribution<Cost> draw(cost_min, cost_max);
  CompGraph::Builder b;
  for (std::size_t i = 0; i < n; ++i) b.add_vertex("v" + std::to_string(i + 1), draw(rng));
  bool edged = false;
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = i + 1; j < n; ++j)
      if (coin(rng) < p) {
        b.add_edge(static_cast<VertexId>(i), static_cast<VertexId>(j));
        edged = true;
      }
  if (!edged && n > 1)
    for (std::size_t i = 0; i + 1 < n; ++i) b.add_edge(static_cast<VertexId>(i), static_cast<VertexId>(i + 1));
  return CompGraph::build(std::move(b));
}

}  // namespace reforward
