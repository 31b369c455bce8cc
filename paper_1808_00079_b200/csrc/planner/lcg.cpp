// Linear computation graphs: §4 Case (1) closed form and Algorithm 1
// (accessibility graph + node-weighted shortest path per candidate max term).
// Behaviour follows reference proj/include/reforward/lcg.hpp:13-188.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "reforward_b200/planner.hpp"

namespace reforward {

Rational Rational::make(std::int64_t n, std::int64_t d) {
  const std::int64_t g = std::gcd(n, d);
  return {n / g, d / g};
}

// k evenly spaced checkpoints on n unit vertices cost k/n + 1/k; the integer
// optimum is one of floor/ceil(sqrt n), the smaller k winning ties.
AnalyticUniform analytic_uniform(std::int64_t n) {
  auto rel = [n](std::int64_t k) { return Rational::make(k * k + n, n * k); };
  std::int64_t r = static_cast<std::int64_t>(std::sqrt(static_cast<double>(n)));
  while (r * r > n) --r;
  while ((r + 1) * (r + 1) <= n) ++r;
  r = std::max<std::int64_t>(r, 1);
  const std::int64_t up = (r * r == n) ? r : r + 1;
  const Rational a = rel(r), b = rel(up);
  if (b.num * a.den < a.num * b.den) return {up, b};
  return {r, a};
}

namespace {

std::vector<Cost> chain_prefix(const CompGraph& chain, const std::vector<VertexId>& order) {
  std::vector<Cost> pre(order.size() + 1, 0);
  for (std::size_t i = 0; i < order.size(); ++i) pre[i + 1] = pre[i] + chain.cost(order[i]);
  return pre;
}

}  // namespace

AccessibilityGraph build_accessibility_graph(const CompGraph& chain, Cost max_term) {
  AccessibilityGraph ag;
  ag.chain = chain.topo_order();  // a chain's topological order is the path
  ag.max_term = max_term;
  ag.prefix = chain_prefix(chain, ag.chain);
  const auto m = static_cast<std::uint32_t>(ag.chain.size());
  for (std::uint32_t i = 0; i + 1 < m; ++i)
    for (std::uint32_t j = i + 1; j < m; ++j)
      if (ag.between(i, j) <= max_term) ag.edges.emplace_back(i, j);
  return ag;
}

// Single forward sweep over positions: label j holds the cheapest way to reach
// j (sum of stored interior costs), then the fewest hops, then the
// lexicographically smallest list of stored positions.
LcgSolution shortest_stored_path(const CompGraph& chain, const AccessibilityGraph& ag) {
  const std::size_t m = ag.chain.size();
  struct Label {
    bool reached = false;
    Cost dist = 0;
    std::uint32_t hops = 0;
    std::vector<std::uint32_t> path;
  };
  std::vector<Label> lab(m);
  lab[0].reached = true;
  std::vector<std::vector<std::uint32_t>> into(m);
  for (const auto& e : ag.edges) into[e.second].push_back(e.first);

  for (std::uint32_t j = 1; j < m; ++j) {
    const bool terminal = (j + 1 == m);
    const Cost w = terminal ? 0 : chain.cost(ag.chain[j]);
    Label& cur = lab[j];
    for (std::uint32_t i : into[j]) {
      const Label& from = lab[i];
      if (!from.reached) continue;
      const Cost d = from.dist + w;
      const std::uint32_t h = from.hops + 1;
      bool take = !cur.reached || d < cur.dist;
      if (!take && d == cur.dist) {
        if (h < cur.hops) {
          take = true;
        } else if (h == cur.hops) {
          std::vector<std::uint32_t> p = from.path;
          if (!terminal) p.push_back(j);
          take = p < cur.path;
        }
      }
      if (take) {
        cur.reached = true;
        cur.dist = d;
        cur.hops = h;
        cur.path = from.path;
        if (!terminal) cur.path.push_back(j);
      }
    }
  }

  const Label& end = lab[m - 1];
  LcgSolution sol;
  sol.stored = VertexSet(chain.n_vertices());
  for (auto pos : end.path) sol.stored.set(ag.chain[pos]);
  sol.stored_cost = end.dist;
  Cost worst = 0;
  std::uint32_t from = 0;
  for (auto pos : end.path) {
    worst = std::max(worst, ag.between(from, pos));
    from = pos;
  }
  worst = std::max(worst, ag.between(from, static_cast<std::uint32_t>(m - 1)));
  sol.max_term = worst;
  sol.total = sol.stored_cost + sol.max_term;
  return sol;
}

LcgSolution solve_lcg(const CompGraph& chain) {
  const auto& order = chain.topo_order();
  const auto pre = chain_prefix(chain, order);
  const std::size_t m = order.size();
  std::vector<Cost> bounds{0};
  for (std::size_t i = 0; i + 1 < m; ++i)
    for (std::size_t j = i + 1; j < m; ++j) bounds.push_back(pre[j] - pre[i + 1]);
  std::sort(bounds.begin(), bounds.end());
  bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());

  LcgSolution best;
  bool have = false;
  for (Cost c : bounds) {
    if (have && c > best.total) break;  // a larger bound alone already loses
    LcgSolution s = shortest_stored_path(chain, build_accessibility_graph(chain, c));
    bool better = !have || s.total < best.total;
    if (!better && s.total == best.total) {
      const auto ns = s.stored.count(), nb = best.stored.count();
      better = ns < nb || (ns == nb && VertexSet::compare_lex(s.stored, best.stored) < 0);
    }
    if (better) {
      best = std::move(s);
      have = true;
    }
  }
  return best;
}

}  // namespace reforward
