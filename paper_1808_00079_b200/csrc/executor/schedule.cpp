// Network building, planning (host planner on the tensor graph), the
// re-forward schedule and the arena layouts.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <numeric>
#include <set>
#include <stdexcept>

#include "executor/net.h"
#include "reforward_b200/planner.hpp"

namespace rfx {

const char* op_kind_name(OpKind k) {
  switch (k) {
    case OpKind::Input: return "input";
    case OpKind::Conv: return "conv";
    case OpKind::BN: return "bn";
    case OpKind::BNAddReLU: return "bn_add_relu";
    case OpKind::ReLU: return "relu";
    case OpKind::MaxPool: return "maxpool";
    case OpKind::AvgPool: return "avgpool";
    case OpKind::FC: return "fc";
    case OpKind::Concat: return "concat";
    case OpKind::Loss: return "loss";
    case OpKind::AvgPool2d: return "avgpool2d";
    case OpKind::Linear: return "linear";
  }
  return "?";
}

namespace {
void require(bool ok, const std::string& msg) {
  if (!ok) throw std::invalid_argument(msg);
}
int round8(int c) { return (c + 7) / 8 * 8; }
int round64(int c) { return (c + 63) / 64 * 64; }
}  // namespace

// ============================================================ building
int Net::add_tensor(const std::string& name, int N, int H, int W, int C, DType dt) {
  Tensor t;
  t.name = name;
  t.N = N;
  t.H = H;
  t.W = W;
  t.C = C;
  t.dtype = dt;
  tensors_.push_back(t);
  return (int)tensors_.size() - 1;
}

int Net::add_op(Op op) {
  require(!planned_, "network is frozen once planned");
  const int id = (int)ops_.size();
  for (int t : op.in) {
    require(t >= 0 && t < (int)tensors_.size(), "op input is not a tensor");
    tensors_[t].consumers.push_back(id);
  }
  tensors_[op.out].producer = id;
  ops_.push_back(std::move(op));
  return id;
}

int Net::add_param(const std::string& name, int kind, int op, long count, std::vector<int> shape) {
  Param p;
  p.name = name;
  p.kind = kind;
  p.op = op;
  p.offset = n_params_;
  p.count = count;
  p.shape = std::move(shape);
  n_params_ += (count + 63) / 64 * 64;
  params_.push_back(p);
  return (int)params_.size() - 1;
}

int Net::input(int H, int W, int C) {
  require(input_t_ < 0, "network already has an input");
  in_c_real_ = C;
  input_t_ = add_tensor("input", batch_, H, W, round8(C), DType::BF16);
  Op op;
  op.kind = OpKind::Input;
  op.name = "input";
  op.out = input_t_;
  add_op(op);
  return input_t_;
}

int Net::conv(int x, int cout, int R, int S, int stride, int pad, const std::string& name) {
  return conv2(x, cout, R, S, stride, pad, pad, name);
}

int Net::conv2(int x, int cout, int R, int S, int stride, int pad, int pad_w, const std::string& name) {
  const Tensor& tx = tensors_.at(x);
  require(tx.dtype == DType::BF16, "conv input must be bf16");
  require(cout % 8 == 0, "conv output channels must be a multiple of 8");
  require(pad >= 0 && pad_w >= 0 && pad < R && pad_w < S, "conv padding must be smaller than the filter");
  require(stride == 1 || pad == pad_w, "strided convolutions need square padding");
  const int P = (tx.H + 2 * pad - R) / stride + 1, Q = (tx.W + 2 * pad_w - S) / stride + 1;
  require(P > 0 && Q > 0, "conv output is empty");
  Op op;
  op.kind = OpKind::Conv;
  op.name = name;
  op.in = {x};
  op.R = R;
  op.S = S;
  op.stride = stride;
  op.pad = pad;
  op.pad_w = pad_w;
  op.cin = tx.C;
  op.cin_real = (x == input_t_) ? in_c_real_ : tx.C;
  op.cout = cout;
  op.cpad = round64(tx.C);
  op.coutpad = round64(cout);
  // narrow inputs (the 3-channel image) go through an explicit im2col; a
  // plain 1x1 stride-1 conv reads any channel count directly
  op.explicit_im2col = tx.C < 32 && !(R == 1 && S == 1 && stride == 1 && pad == 0 && pad_w == 0);
  op.kpad = op.explicit_im2col ? round64(R * S * op.cin_real) : 0;
  op.out = add_tensor(name, tx.N, P, Q, cout, DType::BF16);
  const int id = add_op(op);
  const long kw = ops_[id].explicit_im2col ? ops_[id].kpad : (long)R * S * ops_[id].cpad;
  ops_[id].w_param = add_param(name + ".weight", 0, id, (long)cout * kw, {cout, ops_[id].cin_real, R, S});
  return ops_[id].out;
}

static int new_bn_state(std::vector<BNState>& bns, long& n_state, int C) {
  BNState s;
  s.C = C;
  const long c = (C + 63) / 64 * 64;
  s.mean = n_state;
  s.invstd = n_state + c;
  s.scale = n_state + 2 * c;
  s.shift = n_state + 3 * c;
  s.run_mean = n_state + 4 * c;
  s.run_var = n_state + 5 * c;
  s.coef = n_state + 6 * c;
  n_state += 9 * c;
  bns.push_back(s);
  return (int)bns.size() - 1;
}

int Net::bn(int y, bool relu, const std::string& name) {
  const Tensor ty = tensors_.at(y);
  require(ty.dtype == DType::BF16, "bn input must be bf16");
  Op op;
  op.kind = OpKind::BN;
  op.name = name;
  op.in = {y};
  op.k = relu ? 1 : 0;
  op.out = add_tensor(name, ty.N, ty.H, ty.W, ty.C, DType::BF16);
  op.bn = new_bn_state(bns_, n_state_, ty.C);
  const int id = add_op(op);
  ops_[id].w_param = add_param(name + ".weight", 1, id, ty.C, {ty.C});
  ops_[id].b_param = add_param(name + ".bias", 2, id, ty.C, {ty.C});
  return ops_[id].out;
}

int Net::bn_add_relu(int y, int skip, const std::string& name) {
  const Tensor ty = tensors_.at(y);
  const Tensor& ts = tensors_.at(skip);
  require(ty.N == ts.N && ty.H == ts.H && ty.W == ts.W && ty.C == ts.C, "residual shapes differ");
  Op op;
  op.kind = OpKind::BNAddReLU;
  op.name = name;
  op.in = {y, skip};
  op.out = add_tensor(name, ty.N, ty.H, ty.W, ty.C, DType::BF16);
  op.bn = new_bn_state(bns_, n_state_, ty.C);
  const int id = add_op(op);
  ops_[id].w_param = add_param(name + ".weight", 1, id, ty.C, {ty.C});
  ops_[id].b_param = add_param(name + ".bias", 2, id, ty.C, {ty.C});
  return ops_[id].out;
}

int Net::relu(int x, const std::string& name) {
  const Tensor tx = tensors_.at(x);
  Op op;
  op.kind = OpKind::ReLU;
  op.name = name;
  op.in = {x};
  op.out = add_tensor(name, tx.N, tx.H, tx.W, tx.C, DType::BF16);
  add_op(op);
  return tensors_.size() - 1;
}

int Net::maxpool(int x, int k, int stride, int pad, const std::string& name) {
  const Tensor tx = tensors_.at(x);
  const int P = (tx.H + 2 * pad - k) / stride + 1, Q = (tx.W + 2 * pad - k) / stride + 1;
  Op op;
  op.kind = OpKind::MaxPool;
  op.name = name;
  op.in = {x};
  op.k = k;
  op.stride = stride;
  op.pad = pad;
  op.out = add_tensor(name, tx.N, P, Q, tx.C, DType::BF16);
  add_op(op);
  return tensors_.size() - 1;
}

int Net::avgpool(int x, const std::string& name) {
  const Tensor tx = tensors_.at(x);
  Op op;
  op.kind = OpKind::AvgPool;
  op.name = name;
  op.in = {x};
  op.out = add_tensor(name, tx.N, 1, 1, tx.C, DType::BF16);
  add_op(op);
  return tensors_.size() - 1;
}

int Net::avgpool2d(int x, int k, int stride, int pad, const std::string& name) {
  const Tensor tx = tensors_.at(x);
  require(k >= 1 && stride >= 1 && pad >= 0 && 2 * pad <= k, "bad avgpool2d window");
  const int P = (tx.H + 2 * pad - k) / stride + 1, Q = (tx.W + 2 * pad - k) / stride + 1;
  require(P > 0 && Q > 0, "avgpool2d output is empty");
  Op op;
  op.kind = OpKind::AvgPool2d;
  op.name = name;
  op.in = {x};
  op.k = k;
  op.stride = stride;
  op.pad = pad;
  op.out = add_tensor(name, tx.N, P, Q, tx.C, DType::BF16);
  add_op(op);
  return tensors_.size() - 1;
}

// Hidden fully connected layer (VGG / AlexNet classifier): the NHWC input is
// flattened to H*W*C features; bf16 output [N, out] with bias.  The weight's
// canonical (PyTorch) layout is [out][C*H*W]; the GEMM copy is [out][H*W*C].
int Net::linear(int x, int out_features, const std::string& name) {
  const Tensor tx = tensors_.at(x);
  require(tx.dtype == DType::BF16, "linear input must be bf16");
  require(out_features % 8 == 0, "linear output features must be a multiple of 8");
  Op op;
  op.kind = OpKind::Linear;
  op.name = name;
  op.in = {x};
  op.classes = out_features;
  op.lin_h = tx.H;
  op.lin_w = tx.W;
  op.lin_c = tx.C;
  op.cin = tx.H * tx.W * tx.C;
  op.out = add_tensor(name, tx.N, 1, 1, out_features, DType::BF16);
  const int id = add_op(op);
  ops_[id].w_param = add_param(name + ".weight", 5, id, (long)out_features * ops_[id].cin, {out_features, ops_[id].cin});
  ops_[id].b_param = add_param(name + ".bias", 4, id, out_features, {out_features});
  return ops_[id].out;
}

int Net::fc(int x, int classes, const std::string& name) {
  const Tensor tx = tensors_.at(x);
  require(tx.H == 1 && tx.W == 1, "fc input must be pooled [N, C]");
  Op op;
  op.kind = OpKind::FC;
  op.name = name;
  op.in = {x};
  op.classes = classes;
  op.cin = tx.C;
  op.out = add_tensor(name, tx.N, 1, 1, classes, DType::F32);
  const int id = add_op(op);
  ops_[id].w_param = add_param(name + ".weight", 3, id, (long)classes * tx.C, {classes, tx.C});
  ops_[id].b_param = add_param(name + ".bias", 4, id, classes, {classes});
  logits_t_ = ops_[id].out;
  return logits_t_;
}

int Net::concat(int a, int b, const std::string& name) {
  const Tensor ta = tensors_.at(a);
  const Tensor& tbb = tensors_.at(b);
  require(ta.N == tbb.N && ta.H == tbb.H && ta.W == tbb.W, "concat spatial shapes differ");
  Op op;
  op.kind = OpKind::Concat;
  op.name = name;
  op.in = {a, b};
  op.out = add_tensor(name, ta.N, ta.H, ta.W, ta.C + tbb.C, DType::BF16);
  add_op(op);
  return tensors_.size() - 1;
}

int Net::loss(int logits, const std::string& name) {
  require(tensors_.at(logits).dtype == DType::F32, "loss takes fp32 logits");
  Op op;
  op.kind = OpKind::Loss;
  op.name = name;
  op.in = {logits};
  op.classes = tensors_[logits].C;
  op.out = add_tensor(name, 1, 1, 1, 1, DType::F32);
  add_op(op);
  loss_t_ = op.out;
  return loss_t_;
}

// ============================================================ planning
void Net::graph_export(std::vector<std::string>& names, std::vector<long>& costs,
                       std::vector<std::pair<int, int>>& edges) const {
  names.clear();
  costs.clear();
  edges.clear();
  for (const auto& t : tensors_) {
    names.push_back(t.name);
    costs.push_back(t.cost());
  }
  for (const auto& op : ops_)
    for (int i : op.in) edges.emplace_back(i, op.out);
}

namespace {
reforward::CompGraph tensor_graph(const Net& net) {
  std::vector<std::string> names;
  std::vector<long> costs;
  std::vector<std::pair<int, int>> edges;
  net.graph_export(names, costs, edges);
  reforward::CompGraph::Builder b;
  for (size_t i = 0; i < names.size(); ++i) b.add_vertex(names[i], costs[i]);
  for (auto [u, v] : edges) b.add_edge((reforward::VertexId)u, (reforward::VertexId)v);
  auto g = reforward::CompGraph::build(std::move(b));
  if (g.n_vertices() != names.size()) throw std::runtime_error("tensor graph needed virtual endpoints");
  return g;
}
}  // namespace

void Net::plan_with_stored(const std::vector<char>& stored, const std::string& label) {
  require(input_t_ >= 0 && loss_t_ >= 0, "network needs an input and a loss before planning");
  auto g = tensor_graph(*this);
  require((int)g.source() == input_t_ && (int)g.sink() == loss_t_, "tensor graph endpoints are not input/loss");
  reforward::VertexSet vs(g.n_vertices());
  for (size_t t = 0; t < stored.size(); ++t)
    if (stored[t] && g.is_interior((reforward::VertexId)t)) vs.set(t);
  auto sol = reforward::objective_of(g, vs);
  plan_ = Plan{};
  plan_.policy = label;
  plan_.stored.assign(tensors_.size(), 0);
  plan_.seg_of.assign(tensors_.size(), -1);
  for (auto v : sol.stored.to_indices()) plan_.stored[v] = 1;
  for (size_t s = 0; s < sol.segments.size(); ++s) {
    for (auto v : sol.segments[s].members.to_indices()) plan_.seg_of[v] = (int)s;
    plan_.seg_cost.push_back(sol.segments[s].cost);
  }
  plan_.stored_cost = sol.stored_cost;
  plan_.max_seg = sol.realized_max;
  plan_.total = sol.total;
  plan_.store_all_total = g.interior_total();
  planned_ = true;
  build_schedule();
  layout();
}

void Net::plan(const std::string& policy) {
  require(input_t_ >= 0 && loss_t_ >= 0, "network needs an input and a loss before planning");
  auto g = tensor_graph(*this);
  reforward::Solution sol;
  if (policy == "reforward") {
    sol = reforward::solve_acg(g);
  } else if (policy == "store_all") {
    sol = reforward::store_all(g);
  } else if (policy == "lcg") {
    require(reforward::is_linear_chain(g), "lcg policy needs a linear network");
    auto l = reforward::solve_lcg(g);
    sol = reforward::objective_of(g, l.stored);
  } else if (policy == "sqrt") {
    sol = reforward::sqrt_heuristic_chain(g);
  } else {
    require(false, "unknown policy '" + policy + "'");
  }
  std::vector<char> stored(tensors_.size(), 0);
  for (auto v : sol.stored.to_indices()) stored[v] = 1;
  plan_with_stored(stored, policy);
  plan_.candidate_max_term = sol.candidate_max_term;
}

// ============================================================ schedule
// Tensors an op's backward reads (besides the incoming gradient).
static std::vector<int> backward_needs(const Op& op) {
  switch (op.kind) {
    case OpKind::Conv: return {op.in[0]};
    case OpKind::BN: return {op.in[0]};
    case OpKind::BNAddReLU: return {op.in[0], op.out};
    case OpKind::ReLU: return {op.out};
    case OpKind::MaxPool: return {op.in[0], op.out};
    case OpKind::FC: return {op.in[0]};
    case OpKind::Linear: return {op.in[0]};
    case OpKind::Loss: return {op.in[0]};
    default: return {};
  }
}

void Net::build_schedule() {
  const int nt = (int)tensors_.size(), no = (int)ops_.size();
  sched_.clear();
  for (auto& op : ops_) op.bstat_resident = false;
  std::vector<char> computed(nt, 0), ever(no, 0);
  computed[input_t_] = 1;
  int live_seg = -1;
  long live = 0, peak = 0;
  long reforwards = 0, loads = 0;
  std::vector<std::vector<int>> seg_members(plan_.seg_cost.size());
  for (int t = 0; t < nt; ++t)
    if (plan_.seg_of[t] >= 0) seg_members[plan_.seg_of[t]].push_back(t);  // ascending id = topological

  auto release = [&](int s) {
    if (s < 0) return;
    for (int t : seg_members[s])
      if (computed[t]) {
        computed[t] = 0;
        live -= tensors_[t].cost();
      }
    sched_.push_back({InstrKind::Release, -1, s, false});
  };
  auto emit_forward = [&](int o) {
    const int t = ops_[o].out;
    const bool again = ever[o] != 0;
    sched_.push_back({InstrKind::Forward, o, plan_.seg_of[t], again});
    if (again) ++reforwards;
    ever[o] = 1;
    computed[t] = 1;
    if (t != loss_t_) live += tensors_[t].cost();
    peak = std::max(peak, live);
  };
  // make tensor t valid, re-forwarding inside its segment as needed.  Inputs
  // of an unstored tensor are stored (always resident) or in its own segment.
  std::function<void(int)> ensure = [&](int t) {
    if (computed[t]) return;
    const int s = plan_.seg_of[t];
    if (s >= 0 && s != live_seg) {
      release(live_seg);
      live_seg = s;
      ++loads;
    }
    const Op& op = ops_[tensors_[t].producer];
    for (int i : op.in) ensure(i);
    emit_forward(tensors_[t].producer);
  };

  // ---- first forward: list scheduling over tasks whose inputs are resident,
  // preferring tasks that keep the live segment (stored outputs, or outputs
  // in the live segment) so a segment is finished before the next one starts.
  //
  // A two-input op (residual add, concat) whose output is stored may have its
  // inputs in two different segments, which can never be co-resident in the
  // single re-forward region.  Such an op runs as two phases, each reading one
  // input and writing the stored output slot: add = (1) out <- skip, (2) out <-
  // relu(bn(y) + out); concat = one channel slice per phase.  Phase 1 of the
  // add is an exact bf16 copy, so the result is bit-identical to one pass.
  {
    struct Task {
      int op, phase;  // phase 0 = whole op
    };
    std::vector<Task> tasks;
    for (int o = 0; o < no; ++o) {
      const Op& op = ops_[o];
      if (op.kind == OpKind::Input) continue;
      bool split = false;
      if ((op.kind == OpKind::BNAddReLU || op.kind == OpKind::Concat) && plan_.seg_of[op.out] < 0) {
        const int s0 = plan_.seg_of[op.in[0]], s1 = plan_.seg_of[op.in[1]];
        split = s0 >= 0 && s1 >= 0 && s0 != s1;
      }
      if (split) {
        tasks.push_back({o, 1});
        tasks.push_back({o, 2});
      } else {
        tasks.push_back({o, 0});
      }
    }
    auto task_inputs = [&](const Task& t) -> std::vector<int> {
      const Op& op = ops_[t.op];
      if (t.phase == 0) return op.in;
      if (op.kind == OpKind::BNAddReLU) return {t.phase == 1 ? op.in[1] : op.in[0]};
      return {op.in[t.phase - 1]};
    };
    std::vector<char> tdone(tasks.size(), 0);
    std::vector<int> phases_left(no, 0);
    for (const auto& t : tasks) ++phases_left[t.op];
    size_t left = tasks.size();
    while (left > 0) {
      int keep = -1, sw = -1, first = -1;
      for (size_t k = 0; k < tasks.size(); ++k) {
        if (tdone[k]) continue;
        const Task& t = tasks[k];
        // inputs' producers must be finished; the add's phase 2 after phase 1
        bool order_ok = !(t.phase == 2 && ops_[t.op].kind == OpKind::BNAddReLU && !tdone[k - 1]);
        for (int i : task_inputs(t)) order_ok = order_ok && phases_left[tensors_[i].producer] == 0;
        if (!order_ok) continue;
        if (first < 0) first = (int)k;
        bool ready = true;
        for (int i : task_inputs(t)) ready = ready && computed[i];
        if (!ready) continue;
        const int s = plan_.seg_of[ops_[t.op].out];
        if (s < 0 || s == live_seg) {
          keep = (int)k;
          break;
        }
        if (sw < 0) sw = (int)k;
      }
      const int pick = keep >= 0 ? keep : (sw >= 0 ? sw : first);
      if (pick < 0) throw std::runtime_error("forward schedule deadlock");
      const Task& t = tasks[pick];
      if (t.phase == 0) {
        ensure(ops_[t.op].out);
      } else {
        for (int i : task_inputs(t)) ensure(i);
        const int out = ops_[t.op].out;
        sched_.push_back({InstrKind::Forward, t.op, -1, false, t.phase});
        if (!computed[out]) {
          computed[out] = 1;
          live += tensors_[out].cost();
          peak = std::max(peak, live);
        }
        ever[t.op] = 1;
      }
      tdone[pick] = 1;
      --phases_left[t.op];
      --left;
    }
  }
  rep_.forward_ops = (long)sched_.size();

  // ---- backward: list scheduling on gradient readiness, preferring the live segment
  std::vector<int> pending(nt, 0);
  for (int t = 0; t < nt; ++t) pending[t] = (int)tensors_[t].consumers.size();
  std::vector<char> done(no, 0);
  int remaining = 0;
  for (int o = 0; o < no; ++o)
    if (ops_[o].kind != OpKind::Input) ++remaining;
  auto seg_needed = [&](int o) {
    int s = -1;
    for (int t : backward_needs(ops_[o]))
      if (plan_.seg_of[t] >= 0) {
        if (s >= 0 && s != plan_.seg_of[t]) throw std::runtime_error("op backward spans two segments");
        s = plan_.seg_of[t];
      }
    return s;
  };
  // A tensor read by several ops receives one gradient contribution from each
  // consumer's backward, accumulated in place in bf16 -- which is not
  // associative.  So consumers run their backward in a fixed order (highest
  // op id first) whatever the plan: re-forward and store-all form every
  // gradient sum in the same order and stay bit-identical.  The highest-id
  // remaining op is always eligible, so this cannot deadlock.
  static const bool fixed_order = !std::getenv("RFK_BWD_ORDER") || std::atoi(std::getenv("RFK_BWD_ORDER")) != 0;
  auto order_ok = [&](int o) {
    if (!fixed_order) return true;  // diagnostics only: plan-dependent sums
    for (int i : ops_[o].in)
      for (int c : tensors_[i].consumers)
        if (c > o && !done[c]) return false;
    return true;
  };
  long bwd = 0;
  while (remaining > 0) {
    int pick = -1, pick_any = -1;
    for (int o = no - 1; o >= 0; --o) {
      if (done[o] || ops_[o].kind == OpKind::Input || pending[ops_[o].out] != 0 || !order_ok(o)) continue;
      if (pick_any < 0) pick_any = o;
      const int s = seg_needed(o);
      if (s < 0 || s == live_seg) {
        pick = o;
        break;
      }
    }
    if (pick < 0) pick = pick_any;
    if (pick < 0) throw std::runtime_error("backward schedule deadlock");
    const int s = seg_needed(pick);
    if (s >= 0) {
      bool full = s == live_seg;
      if (full)
        for (int t : seg_members[s]) full = full && computed[t];
      if (!full) {
        if (s != live_seg) {
          release(live_seg);
          live_seg = s;
          ++loads;
        }
        for (int t : seg_members[s]) ensure(t);  // whole segment, topological order
      }
    }
    for (int t : backward_needs(ops_[pick]))
      if (!computed[t]) ensure(t);
    sched_.push_back({InstrKind::Backward, pick, s, false});
    // a conv whose input is a BN's output: is that BN's input resident now?
    // (its dgrad epilogue can then produce the BN's backward statistics)
    if (ops_[pick].kind == OpKind::Conv) {
      const int bp = tensors_[ops_[pick].in[0]].producer;
      if (bp >= 0 && ops_[bp].kind == OpKind::BN) ops_[bp].bstat_resident = computed[ops_[bp].in[0]] != 0;
    }
    ++bwd;
    done[pick] = 1;
    --remaining;
    for (int i : ops_[pick].in) --pending[i];
  }
  release(live_seg);
  rep_.backward_ops = bwd;
  rep_.reforward_ops = reforwards;
  rep_.segment_loads = loads;
  rep_.tracked_peak = peak;
  rep_.planned_total = plan_.total;
  rep_.stored_cost = plan_.stored_cost;
  rep_.max_segment = plan_.max_seg;
  rep_.store_all_total = plan_.store_all_total;
}

// ============================================================ layout
namespace {
// Split-K for a bf16-output implicit GEMM (conv fprop / dgrad through TMA
// im2col), from a cost model of gemm.cu: t = waves * (k blocks * c_bn + per-tile
// b) plus, when split, the fp32 partial round trip (s * M * N * 4 bytes at ~3
// TB/s) and one extra launch.  c_kb = time per 64-wide K block of one tile
// (0.5 us, sweep-fitted; RFK_SPLIT_KB overrides, diagnostics: the per-width
// values of the late-round-2 timelines, 0.30 / 0.33 / 0.42 us, measured
// +0.25 % on ResNet-50).  Outputs of at most 32 channels (DenseNet growth
// convs) never split: their few-K-block partial tiles and the extra finish
// launch cost more than the wave they save (DenseNet-121 8.51 -> 8.36 ms
// without split-K).  Returns {bn, splits}.
std::pair<int, int> im2col_split_plan(long M, int N, long kb) {
  if (const char* e = std::getenv("RFK_NO_SPLITK"); e && std::atoi(e)) return {0, 1};  // diagnostics
  const long mt = (M + 127) / 128;
  double best = -1;
  std::pair<int, int> pick{0, 1};
  for (int bn : {256, 128, 64}) {
    if (bn > 64 && N <= bn / 2) continue;
    const double b = bn == 64 ? 2.5 : (bn == 128 ? 3.5 : 7.0);
    static const double c_kb = std::getenv("RFK_SPLIT_KB") ? std::atof(std::getenv("RFK_SPLIT_KB")) : 0.5;
    for (int s : {1, 2, 3, 4, 6, 8}) {
      if (s > 1 && (kb / s < 6 || N <= 32)) continue;
      const long tiles = mt * ((N + bn - 1) / bn) * s;
      const long waves = (tiles + 147) / 148;
      double t = (double)waves * ((double)((kb + s - 1) / s) * c_kb + b);
      // fp32 partials written and summed once more, plus the finish launch
      static const double bw = std::getenv("RFK_SPLIT_BW") ? std::atof(std::getenv("RFK_SPLIT_BW")) : 3.0e6;
      static const double fixed = std::getenv("RFK_SPLIT_FIXED") ? std::atof(std::getenv("RFK_SPLIT_FIXED")) : 3.0;
      if (s > 1) t += (double)s * M * N * 4.0 / bw + fixed;
      if (best < 0 || t < best - 1e-9) {
        best = t;
        pick = {bn, s};
      }
    }
  }
  return pick;
}

}  // namespace

// Sub-pixel classes of a strided conv's data gradient along one dimension:
// input positions h = s*m + a get taps r = r0 + j*s (j < J) of dy rows
// m + c - j, i.e. a stride-1 correlation over dy with J taps and low padding
// J - 1 - c, over ceil((H - a) / s) output rows.
SubpixelDim subpixel_dim(int a, int stride, int R, int pad, int H) {
  SubpixelDim d;
  d.r0 = (a + pad) % stride;
  d.J = d.r0 < R ? (R - d.r0 + stride - 1) / stride : 0;
  d.c = (a + pad) / stride;
  d.pad_lo = d.J - 1 - d.c;
  d.rows = a < H ? (H - a + stride - 1) / stride : 0;
  return d;
}

// Use the sub-pixel form for a strided k x k dgrad when every class is a
// proper stride-1 correlation and each class GEMM still fills the GPU
// (RFK_SUBPIXEL=0 keeps zero insertion everywhere, 2 forces the sub-pixel
// form regardless of size -- tests).
bool Net::subpixel_ok(const Op& op, const Tensor& x) const {
  const int mode = std::getenv("RFK_SUBPIXEL") ? std::atoi(std::getenv("RFK_SUBPIXEL")) : 1;
  if (mode == 0 || op.stride < 2 || (op.R == 1 && op.S == 1) || op.explicit_im2col || op.in[0] == input_t_) return false;
  for (int a = 0; a < op.stride; ++a) {
    const SubpixelDim h = subpixel_dim(a, op.stride, op.R, op.pad, x.H), w = subpixel_dim(a, op.stride, op.S, op.pad_w, x.W);
    if (h.pad_lo < 0 || w.pad_lo < 0) return false;
  }
  const long class_rows = x.rows() / ((long)op.stride * op.stride);
  const long tiles = (class_rows + 127) / 128 * ((op.cin + 127) / 128);
  // one stream: each class must fill a wave (measured: at 98 tiles, ResNet-50
  // layer3, four serial launches lose); stride 2 with the classes on four
  // parallel streams: the four together must
  const bool par = op.stride == 2 && (!std::getenv("RFK_SUBPIXEL_PAR") || std::atoi(std::getenv("RFK_SUBPIXEL_PAR")) != 0);
  return mode == 2 || (par ? tiles * 4 >= 96 : tiles >= 148);
}

namespace {
// explicit-im2col chunk size (RFK_IM2COL_CHUNK_MB; default 0 = whole batch,
// the fastest measured; chunks trade ~130 MB of workspace for launches)
long im2col_chunk_bytes() {
  const char* e = std::getenv("RFK_IM2COL_CHUNK_MB");
  const long mb = e ? std::atol(e) : 0;
  return mb > 0 ? mb << 20 : (1L << 62);
}

// split-K of a weight-gradient GEMM: enough splits for about one persistent
// wave (148 CTAs), each split keeping >= 8 K blocks (RFK_WG_SPLIT_CAP caps it)
int wgrad_splits(long tiles, long kblocks) {
  // as many K splits as keep tiles x splits within ONE wave of 148 CTAs: a
  // ceil here made e.g. 3 tiles x 50 splits = 150 units, so two CTAs ran a
  // second unit and the launch took two unit times
  long s = std::max(1L, 148 / std::max(1L, tiles));
  // at least kMinKb K blocks per split (RFK_WG_MIN_KB, diagnostics)
  static const long min_kb = std::getenv("RFK_WG_MIN_KB") ? std::atol(std::getenv("RFK_WG_MIN_KB")) : 8;
  s = std::min(s, std::max(1L, kblocks / std::max(1L, min_kb)));
  static const long cap = std::getenv("RFK_WG_SPLIT_CAP") ? std::atol(std::getenv("RFK_WG_SPLIT_CAP")) : 148;
  return (int)std::max(1L, std::min(s, cap));
}
}  // namespace

void Net::layout() {
  const int nt = (int)tensors_.size();
  // activation arena: stored slots, then the shared segment region
  slot_.assign(nt, -1);
  long off = 0;
  for (int t = 0; t < nt; ++t)
    if (plan_.stored[t]) {
      slot_[t] = off;
      off += tensors_[t].cost();
    }
  const long seg_base = off;
  std::vector<long> seg_fill(plan_.seg_cost.size(), 0);
  for (int t = 0; t < nt; ++t)
    if (plan_.seg_of[t] >= 0) {
      slot_[t] = seg_base + seg_fill[plan_.seg_of[t]];
      seg_fill[plan_.seg_of[t]] += tensors_[t].cost();
    }
  arena_bytes_ = seg_base + plan_.max_seg;
  rep_.arena_bytes = arena_bytes_;

  // gradient arena: liveness over the backward instruction order
  const int no = (int)ops_.size();
  std::vector<int> bpos(no, -1);
  int idx = 0;
  for (const auto& ins : sched_)
    if (ins.kind == InstrKind::Backward) bpos[ins.op] = idx++;
  grad_slot_.assign(nt, -1);
  grad_acc_base_.assign(no, 0);
  grad_acc_.clear();
  for (int o = 0; o < no; ++o) {
    grad_acc_base_[o] = (int)grad_acc_.size();
    grad_acc_.resize(grad_acc_.size() + ops_[o].in.size(), 0);
  }
  struct Iv {
    int t, start, end;
    long size;
  };
  std::vector<Iv> ivs;
  std::vector<int> conv_bpos;  // backward positions of the conv backwards, ascending
  for (int o = 0; o < no; ++o)
    if (ops_[o].kind == OpKind::Conv && bpos[o] >= 0) conv_bpos.push_back(bpos[o]);
  std::sort(conv_bpos.begin(), conv_bpos.end());
  const int grad_slack = std::getenv("RFK_GRAD_SLACK") ? std::atoi(std::getenv("RFK_GRAD_SLACK")) : 0;
  for (int t = 0; t < nt; ++t) {
    if (t == input_t_ || t == loss_t_) continue;
    int start = 1 << 30;
    std::vector<std::pair<int, std::pair<int, int>>> writers;  // (bpos, (op, input idx))
    for (int c : tensors_[t].consumers) {
      const Op& op = ops_[c];
      for (size_t i = 0; i < op.in.size(); ++i)
        if (op.in[i] == t) writers.push_back({bpos[c], {c, (int)i}});
    }
    std::sort(writers.begin(), writers.end());
    for (size_t k = 0; k < writers.size(); ++k) {
      grad_acc_[grad_acc_base_[writers[k].second.first] + writers[k].second.second] = k > 0 ? 1 : 0;
      start = std::min(start, writers[k].first);
    }
    int end = bpos[tensors_[t].producer];
    if (writers.empty() || end < 0) continue;
    // a conv's output gradient is read by its weight-gradient GEMM on the side
    // stream after the conv's backward: keep the slot until `slack` further
    // conv backwards have been issued, so the next writers of the gradient
    // arena do not force a join right behind the fork (the gradient arena is
    // not part of Eq. 1; its size is reported separately)
    if (ops_[tensors_[t].producer].kind == OpKind::Conv && wgrad_overlap() && grad_slack > 0) {
      const auto it = std::upper_bound(conv_bpos.begin(), conv_bpos.end(), end);
      const long k = (it - conv_bpos.begin()) + grad_slack - 1;
      end = k < (long)conv_bpos.size() ? conv_bpos[k] : idx;
    }
    ivs.push_back({t, start, end, tensors_[t].cost()});
  }
  std::sort(ivs.begin(), ivs.end(), [](const Iv& a, const Iv& b) { return a.start < b.start || (a.start == b.start && a.t < b.t); });
  std::vector<Iv> active;
  long gpeak = 0;
  for (const auto& iv : ivs) {
    if (!keep_grads_)  // debug mode keeps every gradient tensor in its own slot
      active.erase(std::remove_if(active.begin(), active.end(), [&](const Iv& a) { return a.end < iv.start; }),
                   active.end());
    std::vector<std::pair<long, long>> used;
    for (const auto& a : active) used.push_back({grad_slot_[a.t], grad_slot_[a.t] + a.size});
    std::sort(used.begin(), used.end());
    long pos = 0;
    for (auto [b, e] : used) {
      if (pos + iv.size <= b) break;
      pos = std::max(pos, e);
    }
    grad_slot_[iv.t] = pos;
    gpeak = std::max(gpeak, pos + iv.size);
    active.push_back(iv);
  }
  grad_bytes_ = gpeak;
  rep_.grad_arena_bytes = grad_bytes_;

  // workspaces
  ws_im2col_ = ws_partials_ = ws_zero_ = ws_split_ = ws_stats_ = ws_misc_ = ws_dsplit_ = 0;
  for (auto& op : ops_) {
    if (op.kind == OpKind::Conv) {
      const Tensor& x = tensors_[op.in[0]];
      const Tensor& y = tensors_[op.out];
      if (op.explicit_im2col) {
        // the im2col matrix is built and consumed in chunks of whole images
        // small enough to stay in L2 (the full stem matrix is ~150 MB at
        // batch 32, HBM traffic twice over)
        const long per_img = (long)y.H * y.W * op.kpad * 2;
        op.im2col_imgs = (int)std::max(1L, std::min((long)y.N, im2col_chunk_bytes() / per_img));
        ws_im2col_ = std::max(ws_im2col_, align_up(op.im2col_imgs * per_img));
      }
      const long kw = op.explicit_im2col ? op.kpad : (long)op.R * op.S * op.cpad;
      op.wg_bn = kw <= 64 ? 64 : (kw <= 128 ? 128 : 256);
      const long tiles = ((op.cout + 127) / 128) * ((kw + op.wg_bn - 1) / op.wg_bn);
      if (op.explicit_im2col) {
        // one set of split-K partials per image chunk, summed together (chunk
        // major, split minor) by one reduction
        const long chunks = (y.N + op.im2col_imgs - 1) / op.im2col_imgs;
        op.wg_splits = wgrad_splits(tiles, ((long)op.im2col_imgs * y.H * y.W + 63) / 64);
        ws_split_ = std::max(ws_split_, align_up(chunks * op.wg_splits * op.cout * kw * 4));
      } else {
        op.wg_splits = wgrad_splits(tiles, (y.rows() + 63) / 64);
        if (op.wg_splits > 1) ws_split_ = std::max(ws_split_, align_up((long)op.wg_splits * op.cout * kw * 4));
      }
      // fprop / dgrad through TMA im2col: split-K when the output tiles are
      // too few to fill the GPU (the deep 14x14 / 7x7 layers)
      op.fp_splits = op.dg_splits = 1;
      op.fp_bn = op.dg_bn = 0;
      const bool im2col_fwd = !op.explicit_im2col && !(op.R == 1 && op.S == 1 && op.stride == 1 && op.pad == 0 &&
                                                        op.pad_w == 0);
      if (im2col_fwd && op.cout % 4 == 0 && op.cout / 4 <= 256) {
        const auto pl = im2col_split_plan(y.rows(), op.cout, (long)op.R * op.S * (op.cpad / 64));
        if (pl.second > 1) {
          op.fp_bn = pl.first;
          op.fp_splits = pl.second;
          ws_dsplit_ = std::max(ws_dsplit_, align_up((long)pl.second * y.rows() * op.cout * 4));
        }
      }
      op.dg_subpixel = subpixel_ok(op, x);
      // zero-insertion buffer of a strided k x k data gradient: only where the
      // dgrad exists (not for a conv on the network input, e.g. the stem --
      // 205 MB at batch 32 otherwise) and does not use the sub-pixel classes
      if (op.stride > 1 && !(op.R == 1 && op.S == 1) && op.in[0] != input_t_ && !op.explicit_im2col &&
          !op.dg_subpixel)
        ws_zero_ = std::max(ws_zero_, align_up((long)x.N * (x.H - op.R + 1 + 2 * op.pad) *
                                               (x.W - op.S + 1 + 2 * op.pad_w) * op.cout * 2));
      const bool dgrad_taps = !op.dg_subpixel && op.in[0] != input_t_ && !op.explicit_im2col && !(op.R == 1 && op.S == 1 &&
                                                                                op.pad == 0 && op.pad_w == 0);
      if (dgrad_taps && op.cin % 4 == 0 && op.cin / 4 <= 256) {
        const auto pl = im2col_split_plan(x.rows(), op.cin, (long)op.R * op.S * (op.coutpad / 64));
        if (pl.second > 1) {
          op.dg_bn = pl.first;
          op.dg_splits = pl.second;
          ws_dsplit_ = std::max(ws_dsplit_, align_up((long)pl.second * x.rows() * op.cin * 4));
        }
      }
      // fused BN statistics slot for this conv
      bool fuse = tensors_[op.out].consumers.size() == 1;
      if (fuse) {
        const Op& c = ops_[tensors_[op.out].consumers[0]];
        fuse = (c.kind == OpKind::BN || c.kind == OpKind::BNAddReLU) && c.in[0] == op.out;
      }
      op.fuse_stats = fuse;
    }
    if (op.kind == OpKind::BN || op.kind == OpKind::BNAddReLU) {
      const Tensor& y = tensors_[op.in[0]];
      ws_partials_ = std::max(ws_partials_, align_up((long)rfk::colstats_blocks(y.rows()) * 2 * y.C * 4));
    }
    if (op.kind == OpKind::FC) ws_misc_ = std::max(ws_misc_, align_up((long)batch_ * round8(op.classes) * 2));
    if (op.kind == OpKind::MaxPool)  // window argmax bytes for the backward (shares the zero-insert region)
      ws_zero_ = std::max(ws_zero_, align_up(tensors_[op.out].elems()));
  }
  // BN over a concatenation (DenseNet's BN-ReLU-conv on the growing feature
  // stack): the per-channel batch statistics of a channel do not depend on
  // which concat it sits in, so every leaf tensor's sums are produced once --
  // by its conv's epilogue or one colstats pass after its producer -- and each
  // BN gathers its channels' rows instead of re-reading the whole stack.
  gather_leaves_.clear();
  leaf_stats_off_.assign(tensors_.size(), -1);
  std::vector<char> colstats_leaf(tensors_.size(), 0);
  const bool gather_on = !std::getenv("RFK_BN_GATHER") || std::atoi(std::getenv("RFK_BN_GATHER")) != 0;
  for (auto& op : ops_) {
    op.bn_gather = -1;
    if (!gather_on || (op.kind != OpKind::BN && op.kind != OpKind::BNAddReLU)) continue;
    const int t = op.in[0];
    if (tensors_[t].producer < 0 || ops_[tensors_[t].producer].kind != OpKind::Concat) continue;
    std::vector<int> leaves, stack{t};
    while (!stack.empty()) {  // depth-first, left input first: channel order
      const int u = stack.back();
      stack.pop_back();
      const int pr = tensors_[u].producer;
      if (pr >= 0 && ops_[pr].kind == OpKind::Concat) {
        stack.push_back(ops_[pr].in[1]);
        stack.push_back(ops_[pr].in[0]);
      } else {
        leaves.push_back(u);
      }
    }
    bool ok = true;
    for (int u : leaves) ok = ok && u != input_t_ && tensors_[u].producer >= 0 && tensors_[u].C % 32 == 0;
    if (!ok) continue;
    for (int u : leaves) {
      Op& pr = ops_[tensors_[u].producer];
      if (pr.kind == OpKind::Conv && pr.out == u && !pr.explicit_im2col) pr.fuse_stats = true;
      else colstats_leaf[u] = 1;
    }
    op.bn_gather = (int)gather_leaves_.size();
    gather_leaves_.push_back(std::move(leaves));
  }
  // Re-forward fusion: a conv whose only consumer is a plain BN in the same
  // segment applies that BN (statistics of the first forward) in its own
  // epilogue when both are re-forwarded; the BN's re-forward is then a no-op.
  for (auto& op : ops_) {
    op.fused_bn = -1;
    op.reforward_in_producer = false;
  }
  for (int o = 0; o < (int)ops_.size(); ++o) {
    Op& op = ops_[o];
    if (op.kind != OpKind::Conv || !op.fuse_stats || op.fp_splits > 1) continue;
    const int b = tensors_[op.out].consumers[0];
    Op& bn = ops_[b];
    if (bn.kind != OpKind::BN || bn.out < 0 || op.cout % 8) continue;
    const int s_y = plan_.seg_of[op.out], s_o = plan_.seg_of[bn.out];
    if (s_y < 0 || s_o != s_y) continue;
    op.fused_bn = b;
    bn.reforward_in_producer = true;
  }
  // BN+ReLU backward statistics from rows (see Op::bstat): eligible when the
  // BN's output feeds exactly one conv; fused into that conv's dgrad when
  // the dgrad is one plain launch (1x1 stride 1, or k x k stride 1 without
  // split-K) and the BN input is resident there, else replayed at the BN's
  // backward over the stored dout with the same tiles
  const bool bstat_on = !std::getenv("RFK_BSTAT") || std::atoi(std::getenv("RFK_BSTAT")) != 0;
  for (auto& op : ops_) op.bstat_src = -1;
  for (int o = 0; o < (int)ops_.size(); ++o) {
    Op& bn = ops_[o];
    bn.bstat = bn.bstat_fused = false;
    bn.bstat_off = -1;
    if (!bstat_on || bn.kind != OpKind::BN || bn.k != 1) continue;
    const Tensor& yt = tensors_[bn.in[0]];
    static const int min_c = std::getenv("RFK_BSTAT_MINC") ? std::atoi(std::getenv("RFK_BSTAT_MINC")) : 0;
    if (tensors_[bn.out].consumers.size() != 1 || yt.C % 8 || yt.C < min_c) continue;
    const int c = tensors_[bn.out].consumers[0];
    Op& conv = ops_[c];
    if (conv.kind != OpKind::Conv || conv.in[0] != bn.out || conv.explicit_im2col) continue;
    const bool one_by_one = conv.R == 1 && conv.S == 1 && conv.pad == 0 && conv.pad_w == 0;
    const bool fusible = one_by_one ? conv.stride == 1 : (conv.stride == 1 && !conv.dg_subpixel && conv.dg_splits <= 1);
    // (a dgrad that can never fuse keeps the streaming reduction: replaying
    // it through the GEMM epilogue measured slower)
    if (!fusible) continue;
    bn.bstat = true;
    // the rows' tile width: the dgrad's own (auto) choice when it can fuse
    rfk::GemmDesc d;
    d.M = (int)yt.rows();
    d.N = yt.C;
    if (fusible && one_by_one) {
      d.K = conv.cout;
      d.a_kind = rfk::Operand::KMajor2D;
      d.b_kind = rfk::Operand::MNMajor2D;
    } else if (fusible) {
      const Tensor& ct = tensors_[conv.out];
      d.K = conv.R * conv.S * conv.coutpad;
      d.a_kind = rfk::Operand::Im2colK;
      d.a_geom = rfk::ConvGeom{ct.N, ct.H, ct.W, conv.cout, yt.H, yt.W, conv.R, conv.S, conv.R - 1 - conv.pad,
                               conv.S - 1 - conv.pad_w, 1, 1};
      d.b_kind = rfk::Operand::WeightTapsMN;
    } else {
      d.K = 64;
      d.a_kind = rfk::Operand::KMajor2D;
      d.b_kind = rfk::Operand::KMajor2D;
    }
    bn.bstat_bn = rfk::gemm_block_n(d);
    bn.bstat_fused = fusible && bn.bstat_resident;
    if (bn.bstat_fused) conv.bstat_src = o;
    bn.bstat_off = ws_stats_ / 4;  // [kStatRows][2][C], written only by this BN's rows producer
    ws_stats_ += align_up(kStatRows * 2 * (long)yt.C * 4);
  }
  for (auto& op : ops_)
    if (op.kind == OpKind::Conv && op.fuse_stats) {
      op.stats_off = ws_stats_ / 4;  // [kStatRows][2][cout]: one row per persistent GEMM CTA
      ws_stats_ += align_up(kStatRows * 2 * op.cout * 4);
    }
  for (int t = 0; t < (int)tensors_.size(); ++t)
    if (colstats_leaf[t]) {  // [colstats_blocks][2][C]
      leaf_stats_off_[t] = ws_stats_ / 4;
      ws_stats_ += align_up((long)rfk::colstats_blocks(tensors_[t].rows()) * 2 * tensors_[t].C * 4);
    }
  ws_counters_ = 0;
  // max pools keep their argmax from the forward (and every re-forward): the
  // backward gathers dy through it and never re-reads x (RFK_POOL_IDX=0: the
  // fused tiled backward over x instead)
  ws_pool_ = 0;
  const bool pool_idx = !std::getenv("RFK_POOL_IDX") || std::atoi(std::getenv("RFK_POOL_IDX")) != 0;
  for (auto& op : ops_) {
    op.pool_idx_off = -1;
    if (!pool_idx || op.kind != OpKind::MaxPool || op.k * op.k > 256) continue;
    op.pool_idx_off = ws_pool_;
    ws_pool_ += align_up(tensors_[op.out].elems());
  }
  rep_.workspace_bytes =
      ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_ + ws_stats_ + ws_misc_ + ws_counters_ + ws_dsplit_ + ws_pool_;
  if (std::getenv("RFK_TRACE_WS"))
    std::fprintf(stderr, "workspace MB: im2col %.1f partials %.1f zero/argmax %.1f wgrad-split %.1f stats %.1f misc %.1f "
                 "fprop/dgrad-split %.1f\n", ws_im2col_ / 1e6, ws_partials_ / 1e6, ws_zero_ / 1e6, ws_split_ / 1e6,
                 ws_stats_ / 1e6, ws_misc_ / 1e6, ws_dsplit_ / 1e6);
  rep_.param_bytes = n_params_ * 4 * 3;
  rep_.state_bytes = n_state_ * 4;
}

long Net::flops_per_step() const {
  // algorithmic MACs x 2 of the dense contractions: forward + dgrad + wgrad
  long f = 0;
  for (const auto& op : ops_) {
    if (op.kind == OpKind::Conv) {
      const Tensor& y = tensors_[op.out];
      const long fwd = 2L * y.rows() * op.cout * op.R * op.S * op.cin_real;
      const bool dgrad = op.in[0] != input_t_;
      f += fwd * (dgrad ? 3 : 2);
    } else if (op.kind == OpKind::FC || op.kind == OpKind::Linear) {
      f += 2L * batch_ * op.classes * op.cin * 3;
    }
  }
  return f;
}

}  // namespace rfx
