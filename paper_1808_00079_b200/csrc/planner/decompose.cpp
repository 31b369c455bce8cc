// Closed sets (Defs. 1-8, Algorithms 2-4) and the division tree (Def. 9).
// Behaviour follows reference proj/include/reforward/closed_set.hpp:16-408 and
// division_tree.hpp:18-194; the set algebra here is done on reachability /
// adjacency bitsets instead of per-pair scans.
#include <algorithm>

#include "reforward_b200/planner.hpp"

namespace reforward {

const char* to_string(ClosedSetType t) {
  switch (t) {
    case ClosedSetType::Splittable: return "splittable";
    case ClosedSetType::Branched: return "branched";
    case ClosedSetType::NonBranched: return "non-branched";
  }
  return "?";
}

namespace {

// Adjacency inside one closed-set instance: the graph's undirected adjacency,
// except that the entry-exit edge is absent when the instance excludes it.
bool adjacent_in(const CompGraph& g, const ClosedSet& cs, VertexId a, VertexId b) {
  const bool is_pair = (a == cs.entry && b == cs.exit) || (a == cs.exit && b == cs.entry);
  if (is_pair && !cs.includes_direct_edge) return false;
  return g.connected(a, b);
}

VertexSet closure_of(const ClosedSet& cs) {
  VertexSet c = cs.members;
  c.set(cs.entry);
  c.set(cs.exit);
  return c;
}

// Vertices strictly between a and b inside `pool`.
VertexSet between_set(const CompGraph& g, const VertexSet& pool, VertexId a, VertexId b) {
  VertexSet s = pool;
  s &= g.descendants(a);
  s &= g.ancestors(b);
  if (a < s.capacity()) s.reset(a);
  if (b < s.capacity()) s.reset(b);
  return s;
}

bool pair_before(const CompGraph& g, const ClosedSet& x, const ClosedSet& y) {
  const auto xe = g.topo_index(x.entry), ye = g.topo_index(y.entry);
  if (xe != ye) return xe < ye;
  return g.topo_index(x.exit) < g.topo_index(y.exit);
}

// Largest closed set between (k, t) inside `parent`, or the bare direct edge
// when the full candidate touches the rest of the parent (closed_set.hpp:160-188).
std::optional<ClosedSet> closed_set_between(const CompGraph& g, const ClosedSet& parent, VertexId k,
                                            VertexId t) {
  VertexSet inner = between_set(g, parent.members, k, t);
  const bool direct = g.has_edge(k, t) && adjacent_in(g, parent, k, t);
  if (inner.any()) {
    // Property 3 relative to the parent's closure: every neighbour of an
    // inner vertex must be inner or one of the two endpoints.  Inner vertices
    // are parent members, so the parent's entry-exit exception never applies.
    VertexSet allowed = inner;
    allowed.set(k);
    allowed.set(t);
    const VertexSet pc = closure_of(parent);
    bool sealed = true;
    for (auto v : inner.to_indices()) {
      VertexSet leak = g.neighbour_set(v);
      leak &= pc;
      if (!leak.is_subset_of(allowed)) {
        sealed = false;
        break;
      }
    }
    if (sealed) return make_closed_set(g, k, t, std::move(inner), direct);
  }
  if (direct) return make_closed_set(g, k, t, VertexSet(g.n_vertices()), true);
  return std::nullopt;
}

// Edge indices whose both endpoints lie in the set's closure.
VertexSet owned_edges(const CompGraph& g, const ClosedSet& s) {
  const VertexSet c = closure_of(s);
  VertexSet e(g.edges().size());
  for (std::size_t i = 0; i < g.edges().size(); ++i)
    if (c.test(g.edges()[i].first) && c.test(g.edges()[i].second)) e.set(i);
  return e;
}

bool parts_disjoint(const CompGraph& g, const std::vector<ClosedSet>& parts) {
  std::vector<VertexSet> es;
  for (const auto& p : parts) es.push_back(owned_edges(g, p));
  for (std::size_t i = 0; i < parts.size(); ++i)
    for (std::size_t j = i + 1; j < parts.size(); ++j)
      if (parts[i].members.intersects(parts[j].members) || es[i].intersects(es[j])) return false;
  return true;
}

bool parts_cover(const CompGraph& g, const ClosedSet& cs, const std::vector<ClosedSet>& parts) {
  VertexSet vc(g.n_vertices());
  vc.set(cs.entry);
  vc.set(cs.exit);
  VertexSet ec(g.edges().size());
  for (const auto& p : parts) {
    vc |= closure_of(p);
    ec |= owned_edges(g, p);
  }
  return vc == closure_of(cs) && owned_edges(g, cs).is_subset_of(ec);
}

// Edge-only closed sets for every graph edge inside `cs`'s closure except its
// own entry->exit edge, in graph edge order.
std::vector<ClosedSet> edge_atoms(const CompGraph& g, const ClosedSet& cs) {
  const VertexSet c = closure_of(cs);
  std::vector<ClosedSet> atoms;
  for (const auto& [u, v] : g.edges()) {
    if (!c.test(u) || !c.test(v)) continue;
    if (u == cs.entry && v == cs.exit) continue;
    atoms.push_back(make_closed_set(g, u, v, VertexSet(g.n_vertices()), true));
  }
  return atoms;
}

// Undirected components of `members`, seeds taken in topological order.
std::vector<VertexSet> member_components(const CompGraph& g, const VertexSet& members) {
  auto ids = members.to_indices();
  std::sort(ids.begin(), ids.end(), [&](VertexId a, VertexId b) { return g.topo_index(a) < g.topo_index(b); });
  VertexSet done(g.n_vertices());
  std::vector<VertexSet> comps;
  for (VertexId seed : ids) {
    if (done.test(seed)) continue;
    VertexSet comp(g.n_vertices());
    comp.set(seed);
    std::vector<VertexId> todo{seed};
    while (!todo.empty()) {
      VertexId v = todo.back();
      todo.pop_back();
      VertexSet nb = g.neighbour_set(v);
      nb &= members;
      for (auto w : nb.to_indices())
        if (!comp.test(w)) {
          comp.set(w);
          todo.push_back(w);
        }
    }
    done |= comp;
    comps.push_back(std::move(comp));
  }
  return comps;
}

}  // namespace

ClosedSet make_closed_set(const CompGraph& g, VertexId entry, VertexId exit, VertexSet members,
                          bool includes_direct_edge) {
  ClosedSet cs;
  cs.entry = entry;
  cs.exit = exit;
  cs.cost = interior_cost(g, members);
  cs.members = std::move(members);
  cs.includes_direct_edge = includes_direct_edge;
  return cs;
}

ClosedSet whole_graph_set(const CompGraph& g) {
  return make_closed_set(g, g.source(), g.sink(), g.interior(), g.has_edge(g.source(), g.sink()));
}

// Algorithm 2: v splits cs iff every other closure vertex is strictly before
// or strictly after v and no edge of the instance joins the two sides.
bool is_splitting_vertex(const ClosedSet& cs, VertexId v, const CompGraph& g) {
  VertexSet rest = closure_of(cs);
  rest.reset(v);
  VertexSet before = rest, after = rest;
  before &= g.ancestors(v);
  after &= g.descendants(v);
  if (before.intersects(after)) return false;
  VertexSet both = before;
  both |= after;
  if (both != rest) return false;
  for (auto a : before.to_indices()) {
    VertexSet nb = g.neighbour_set(a);
    nb &= after;
    for (auto b : nb.to_indices())
      if (adjacent_in(g, cs, a, b)) return false;
  }
  return true;
}

// Algorithm 3: branched iff the direct edge rides along with members, or the
// members do not form one undirected component.
bool is_branched(const ClosedSet& cs, const CompGraph& g) {
  if (!cs.members.any()) return false;
  if (cs.includes_direct_edge) return true;
  return member_components(g, cs.members).size() > 1;
}

ClosedSetType classify(const ClosedSet& cs, const CompGraph& g) {
  for (auto v : cs.members.to_indices())
    if (is_splitting_vertex(cs, v, g)) return ClosedSetType::Splittable;
  if (is_branched(cs, g)) return ClosedSetType::Branched;
  return ClosedSetType::NonBranched;
}

std::vector<ClosedSet> enumerate_closed_sets(const CompGraph& g) {
  const ClosedSet whole = whole_graph_set(g);
  const auto& ord = g.topo_order();
  std::vector<ClosedSet> found;
  for (std::size_t i = 0; i < ord.size(); ++i)
    for (std::size_t j = i + 1; j < ord.size(); ++j)
      if (auto cs = closed_set_between(g, whole, ord[i], ord[j])) found.push_back(std::move(*cs));
  return found;
}

// Algorithm 4 with the reference's two fallbacks (closed_set.hpp:271-354):
// containment-maximal formed sets; else greedy largest-first packing with
// edge atoms in the pool; else edge atoms alone.
std::vector<ClosedSet> maximal_split(const ClosedSet& cs, const CompGraph& g) {
  auto verts = closure_of(cs).to_indices();
  std::sort(verts.begin(), verts.end(), [&](VertexId a, VertexId b) { return g.topo_index(a) < g.topo_index(b); });

  std::vector<ClosedSet> formed;
  for (std::size_t i = 0; i < verts.size(); ++i)
    for (std::size_t j = i + 1; j < verts.size(); ++j) {
      if (verts[i] == cs.entry && verts[j] == cs.exit) continue;
      if (auto s = closed_set_between(g, cs, verts[i], verts[j])) formed.push_back(std::move(*s));
    }

  std::vector<VertexSet> cl;
  for (const auto& s : formed) cl.push_back(closure_of(s));
  std::vector<ClosedSet> keep;
  for (std::size_t i = 0; i < formed.size(); ++i) {
    bool inside_other = false;
    for (std::size_t j = 0; j < formed.size() && !inside_other; ++j)
      inside_other = j != i && cl[i] != cl[j] && cl[i].is_subset_of(cl[j]);
    if (!inside_other) keep.push_back(formed[i]);
  }
  auto by_pair = [&](const ClosedSet& a, const ClosedSet& b) { return pair_before(g, a, b); };
  std::sort(keep.begin(), keep.end(), by_pair);
  if (parts_disjoint(g, keep) && parts_cover(g, cs, keep)) return keep;

  std::vector<ClosedSet> pool = formed;
  for (auto& a : edge_atoms(g, cs)) pool.push_back(std::move(a));
  std::stable_sort(pool.begin(), pool.end(), [&](const ClosedSet& a, const ClosedSet& b) {
    const auto na = a.members.count(), nb = b.members.count();
    if (na != nb) return na > nb;
    return pair_before(g, a, b);
  });
  std::vector<ClosedSet> packed;
  std::vector<VertexSet> packed_e, packed_c;
  for (const auto& p : pool) {
    const VertexSet pe = owned_edges(g, p), pc = closure_of(p);
    bool fits = true;
    for (std::size_t i = 0; fits && i < packed.size(); ++i)
      fits = !pe.intersects(packed_e[i]) && !p.members.intersects(packed_c[i]) &&
             !packed[i].members.intersects(pc);
    if (!fits) continue;
    packed.push_back(p);
    packed_e.push_back(pe);
    packed_c.push_back(pc);
  }
  std::sort(packed.begin(), packed.end(), by_pair);
  if (parts_disjoint(g, packed) && parts_cover(g, cs, packed)) return packed;

  auto atoms = edge_atoms(g, cs);
  std::sort(atoms.begin(), atoms.end(), by_pair);
  return atoms;
}

std::vector<ClosedSet> divide(const ClosedSet& cs, const CompGraph& g) {
  std::vector<VertexId> cut;
  for (auto v : cs.members.to_indices())
    if (is_splitting_vertex(cs, v, g)) cut.push_back(v);

  std::vector<ClosedSet> parts;
  if (!cut.empty()) {
    std::sort(cut.begin(), cut.end(), [&](VertexId a, VertexId b) { return g.topo_index(a) < g.topo_index(b); });
    cut.insert(cut.begin(), cs.entry);
    cut.push_back(cs.exit);
    for (std::size_t i = 0; i + 1 < cut.size(); ++i) {
      const VertexId a = cut[i], b = cut[i + 1];
      const bool direct = g.has_edge(a, b) && adjacent_in(g, cs, a, b);
      parts.push_back(make_closed_set(g, a, b, between_set(g, cs.members, a, b), direct));
    }
    return parts;
  }
  if (is_branched(cs, g)) {
    for (auto& comp : member_components(g, cs.members))
      parts.push_back(make_closed_set(g, cs.entry, cs.exit, std::move(comp), false));
    if (cs.includes_direct_edge)
      parts.push_back(make_closed_set(g, cs.entry, cs.exit, VertexSet(g.n_vertices()), true));
    return parts;
  }
  return maximal_split(cs, g);
}

// ============================================================ division tree
namespace {

std::string quoted_pair(const CompGraph& g, const ClosedSet& s) {
  return "'" + g.name(s.entry) + "' and '" + g.name(s.exit) + "'";
}

// Edges a part owns for ownership accounting: its closure edges, minus its
// own entry->exit edge when the instance excludes it.
VertexSet accounted_edges(const CompGraph& g, const ClosedSet& s) {
  VertexSet e = owned_edges(g, s);
  if (!s.includes_direct_edge)
    for (std::size_t i = 0; i < g.edges().size(); ++i)
      if (g.edges()[i].first == s.entry && g.edges()[i].second == s.exit) e.reset(i);
  return e;
}

// Partition checks of division_tree.hpp:39-86, same messages, same order.
void check_division(const CompGraph& g, const ClosedSet& parent, const std::vector<ClosedSet>& parts) {
  if (parts.empty()) throw DecompositionError("division of set between " + quoted_pair(g, parent) + " is empty");
  VertexSet inner(g.n_vertices()), vc(g.n_vertices());
  vc.set(parent.entry);
  vc.set(parent.exit);
  for (const auto& p : parts) {
    if (p.entry == parent.entry && p.exit == parent.exit && p.members == parent.members &&
        p.includes_direct_edge == parent.includes_direct_edge)
      throw DecompositionError("division returned the set itself between " + quoted_pair(g, parent));
    if (p.members.intersects(inner)) throw DecompositionError("division members overlap");
    inner |= p.members;
    vc |= closure_of(p);
  }
  if (vc != closure_of(parent)) throw DecompositionError("division closures do not cover the set");
  for (const auto& p : parts)
    if (inner.test(p.entry) || inner.test(p.exit))
      throw DecompositionError("division member endpoint buried in an interior");
  VertexSet ec(g.edges().size());
  for (const auto& p : parts) {
    const VertexSet pe = accounted_edges(g, p);
    if (pe.intersects(ec)) throw DecompositionError("division members share an edge");
    ec |= pe;
  }
  if (!accounted_edges(g, parent).is_subset_of(ec))
    throw DecompositionError("division members do not cover all edges");
}

void grow(const CompGraph& g, DivisionTreeNode& node, std::uint32_t& counter) {
  node.id = counter++;
  if (node.kind == DivisionTreeNode::Kind::Vertex || node.set.empty_interior()) return;
  const ClosedSet& cs = node.set;
  node.type = classify(cs, g);
  const auto parts = divide(cs, g);
  check_division(g, cs, parts);
  node.divided = true;

  // Children: the parts plus the boundary vertices they introduce, ordered by
  // (entry rank, exit rank, vertex-before-set, first member rank).
  struct Slot {
    std::size_t k0, k1;
    int vertex_first;  // 0 for a vertex, 1 for a set
    std::size_t k2;
    VertexId v;
    const ClosedSet* part;
  };
  std::vector<Slot> slots;
  VertexSet boundary(g.n_vertices());
  for (const auto& p : parts)
    for (VertexId e : {p.entry, p.exit})
      if (e != cs.entry && e != cs.exit) boundary.set(e);
  for (auto v : boundary.to_indices()) slots.push_back({g.topo_index(v), g.topo_index(v), 0, 0, v, nullptr});
  for (const auto& p : parts) {
    std::size_t first = g.n_vertices() + 1;
    for (auto v : p.members.to_indices()) first = std::min(first, g.topo_index(v));
    slots.push_back({g.topo_index(p.entry), g.topo_index(p.exit), 1, first, 0, &p});
  }
  std::sort(slots.begin(), slots.end(), [](const Slot& a, const Slot& b) {
    if (a.k0 != b.k0) return a.k0 < b.k0;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    if (a.vertex_first != b.vertex_first) return a.vertex_first < b.vertex_first;
    return a.k2 < b.k2;
  });
  for (const auto& s : slots) {
    auto child = std::make_unique<DivisionTreeNode>();
    if (s.part) {
      child->kind = DivisionTreeNode::Kind::Set;
      child->set = *s.part;
    } else {
      child->kind = DivisionTreeNode::Kind::Vertex;
      child->vertex = s.v;
    }
    grow(g, *child, counter);
    node.children.push_back(std::move(child));
  }
}

}  // namespace

std::unique_ptr<DivisionTreeNode> build_division_tree(const CompGraph& g) {
  auto root = std::make_unique<DivisionTreeNode>();
  root->set = whole_graph_set(g);
  std::uint32_t counter = 0;
  grow(g, *root, counter);
  return root;
}

std::size_t count_nodes(const DivisionTreeNode& node) {
  std::size_t n = 1;
  for (const auto& c : node.children) n += count_nodes(*c);
  return n;
}

void dump_tree_text(const CompGraph& g, const DivisionTreeNode& node, std::string& out, int depth) {
  out.append(static_cast<std::size_t>(depth) * 2, ' ');
  if (node.is_vertex_leaf()) {
    out += g.name(node.vertex) + " (tensor, cost " + std::to_string(g.cost(node.vertex)) + ")\n";
    return;
  }
  out += "[" + g.name(node.set.entry) + " .. " + g.name(node.set.exit) + "] cost=" + std::to_string(node.set.cost);
  if (node.divided) out += std::string(" type=") + to_string(node.type);
  else if (node.set.empty_interior()) out += " (edge)";
  out += "\n";
  for (const auto& c : node.children) dump_tree_text(g, *c, out, depth + 1);
}

std::string canonical_form(const CompGraph& g, const DivisionTreeNode& node) {
  if (node.is_vertex_leaf()) return "v:" + std::to_string(g.cost(node.vertex));
  std::vector<std::string> kids;
  for (const auto& c : node.children) kids.push_back(canonical_form(g, *c));
  std::sort(kids.begin(), kids.end());
  std::string s = node.divided ? std::string("n") + to_string(node.type) : std::string("leaf");
  s += ":" + std::to_string(node.set.cost) + "(";
  for (const auto& k : kids) s += k + ",";
  return s + ")";
}

}  // namespace reforward
