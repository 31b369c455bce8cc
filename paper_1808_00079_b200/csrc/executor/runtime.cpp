// Device side of the executor: arenas, parameters, per-op forward/backward
// dispatch onto the sm_100a kernels, SGD, CUDA-graph capture of the step.
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>

#include "executor/comm.h"
#include "executor/net.h"

namespace rfx {

namespace {
int round8(int c) { return (c + 7) / 8 * 8; }

// The shifted-band implicit GEMM (gemm_band.cu) is exact (tests/test_gemm_gpu.py)
// and moves 3-5x fewer A bytes than TMA im2col; it runs where it measured
// faster (gemm_band_preferred: the 56x56 3x3 convs, the narrow DenseNet growth
// convs) and its epilogue suffices (no fused re-forward BN apply, no
// BN-backward statistics).  RFK_BAND=0: never; RFK_BAND=1: wherever allowed.
// sub-pixel class GEMMs on parallel streams (RFK_SUBPIXEL_PAR=0: one stream)
bool sub_parallel() {
  static const bool on = !std::getenv("RFK_SUBPIXEL_PAR") || std::atoi(std::getenv("RFK_SUBPIXEL_PAR")) != 0;
  return on;
}

// A conv that some plan may re-forward with its consumer BN applied in the
// GEMM epilogue (the structural part of the fusion rule in schedule.cpp; which
// plans actually fuse depends on their segments)
bool fusable_conv_impl(const std::vector<Op>& ops, const std::vector<Tensor>& tensors, const Op& op) {
  if (op.kind != OpKind::Conv || !op.fuse_stats || op.fp_splits > 1 || op.cout % 8) return false;
  const auto& cons = tensors[op.out].consumers;
  if (cons.empty()) return false;
  const Op& bn = ops[cons[0]];
  return bn.kind == OpKind::BN && bn.out >= 0;
}

// Stream priorities inside the step graph (RFK_PRIO=1): the capture stream
// (main path: forward, data gradients, BN backward) at the greatest priority,
// the side streams (weight gradients, sub-pixel classes, all-reduce / SGD) at
// the least, so when both have CTAs waiting the critical path goes first; the
// graph is instantiated with node priorities.
// (RFK_PRIO=2: the other way round, side streams first)
int prio_mode() {
  static const int m = std::getenv("RFK_PRIO") ? std::atoi(std::getenv("RFK_PRIO")) : 0;
  return m;
}
bool prio_enabled() { return prio_mode() != 0; }
void create_stream(cudaStream_t* s, bool high) {
  int lo = 0, hi = 0;
  if (prio_enabled() && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess) {
    const bool h = prio_mode() == 2 ? !high : high;
    if (cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, h ? hi : lo) == cudaSuccess) return;
  }
  if (cudaStreamCreateWithFlags(s, cudaStreamNonBlocking) != cudaSuccess) throw std::runtime_error("stream create");
}

int band_enabled() {
  static const int mode = [] {
    const char* e = std::getenv("RFK_BAND");
    return e == nullptr ? 1 : (std::atoi(e) != 0 ? 2 : 0);
  }();
  return mode;
}

float bf16_to_float(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
}  // namespace

bool Net::fusable_conv(const Op& op) const { return fusable_conv_impl(ops_, tensors_, op); }

std::unique_ptr<Net> make_net(int batch) { return std::make_unique<Net>(batch); }

Net::~Net() {
  free_device();
  comm_.reset();
  for (auto e : bucket_events_) cudaEventDestroy(e);
  if (comm_done_) cudaEventDestroy(comm_done_);
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  if (wgrad_fork_) cudaEventDestroy(wgrad_fork_);
  if (wgrad_join_) cudaEventDestroy(wgrad_join_);
  if (wgrad_stream_) cudaStreamDestroy(wgrad_stream_);
  if (sub_fork_) cudaEventDestroy(sub_fork_);
  for (int i = 0; i < 3; ++i) {
    if (sub_join_[i]) cudaEventDestroy(sub_join_[i]);
    if (sub_stream_[i]) cudaStreamDestroy(sub_stream_[i]);
  }
}

void Net::check(cudaError_t e, const char* what) const {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void Net::free_device() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  graph_exec_ = nullptr;
  for (auto& e : phase_exec_) {
    if (e) cudaGraphExecDestroy(e);
    e = nullptr;
  }
  gemm_trace_.clear();
  if (d_prep_table_) cudaFree(d_prep_table_);
  d_prep_table_ = nullptr;
  if (d_gather_) cudaFree(d_gather_);
  d_gather_ = nullptr;
  for (int k = 0; k < 2; ++k) {
    if (d_stage_images_[k]) cudaFree(d_stage_images_[k]);
    if (d_stage_labels_[k]) cudaFree(d_stage_labels_[k]);
    if (stage_ready_[k]) cudaEventDestroy(stage_ready_[k]);
    if (stage_free_[k]) cudaEventDestroy(stage_free_[k]);
    d_stage_images_[k] = nullptr;
    d_stage_labels_[k] = nullptr;
    stage_ready_[k] = stage_free_[k] = nullptr;
  }
  for (void* p : {(void*)d_arena_, (void*)d_grad_arena_, (void*)d_ws_, (void*)d_param_, (void*)d_grad_,
                  (void*)d_mom_, (void*)d_bf16_, (void*)d_state_, (void*)d_input_, (void*)d_images_,
                  (void*)d_labels_, (void*)d_loss_, (void*)d_rowloss_, (void*)d_lse_, (void*)d_hyper_})
    if (p) cudaFree(p);
  d_arena_ = d_grad_arena_ = d_ws_ = nullptr;
  d_param_ = d_grad_ = d_mom_ = d_state_ = d_images_ = d_loss_ = d_rowloss_ = d_lse_ = d_hyper_ = nullptr;
  d_bf16_ = d_input_ = nullptr;
  d_labels_ = nullptr;
  setup_done_ = false;
}

// ============================================================ setup
void Net::setup(uint64_t seed) {
  if (!planned_) throw std::invalid_argument("plan the network before setup");
  free_device();
  // bf16 weight copies
  // the bf16 weight buffer mirrors the fp32 master buffer element for element
  // (BN parameters ride along unused), so refreshing it after SGD is one flat
  // vectorised cast; dgrad reads the same copy through a transposing TMA map
  n_bf16_ = n_params_;
  for (auto& p : params_) {
    p.bf16_off = p.offset;
    p.bf16_count = p.count;
  }
  rep_.device_bytes = 0;
  auto alloc = [&](void** p, long bytes, const char* what) {
    check(cudaMalloc(p, bytes > 0 ? bytes : 256), what);
    rep_.device_bytes += bytes > 0 ? bytes : 256;
  };
  // the activation arena is exactly the planner's Eq. 1 total; a guard band
  // behind it (filled with a canary) lets tests check that no kernel of the
  // step ever writes past that high-water mark
  alloc((void**)&d_arena_, arena_bytes_ + kArenaGuard, "activation arena");
  check(cudaMemset(d_arena_ + arena_bytes_, 0xA5, kArenaGuard), "arena guard");
  alloc((void**)&d_grad_arena_, grad_bytes_, "gradient arena");
  alloc((void**)&d_ws_, rep_.workspace_bytes, "workspace");
  alloc((void**)&d_param_, n_params_ * 4, "params");
  alloc((void**)&d_grad_, n_params_ * 4, "grads");
  alloc((void**)&d_mom_, n_params_ * 4, "momentum");
  alloc((void**)&d_bf16_, n_bf16_ * 2, "bf16 weights");
  alloc((void**)&d_state_, n_state_ * 4, "bn state");
  const Tensor& in = tensors_[input_t_];
  alloc((void**)&d_input_, in.bytes(), "input");
  alloc((void**)&d_images_, (long)batch_ * in_c_real_ * in.H * in.W * 4, "images");
  alloc((void**)&d_labels_, batch_ * 4, "labels");
  alloc((void**)&d_loss_, 256, "loss");
  alloc((void**)&d_rowloss_, batch_ * 4, "row loss");
  alloc((void**)&d_lse_, batch_ * 4, "lse");
  alloc((void**)&d_hyper_, 256, "hyper");
  check(cudaMemset(d_grad_, 0, n_params_ * 4), "memset");
  check(cudaMemset(d_mom_, 0, n_params_ * 4), "memset");
  check(cudaMemset(d_bf16_, 0, n_bf16_ * 2), "memset");
  check(cudaMemset(d_arena_, 0, arena_bytes_ > 0 ? arena_bytes_ : 256), "memset");
  check(cudaMemset(d_ws_, 0, rep_.workspace_bytes > 0 ? rep_.workspace_bytes : 256), "memset");
  check(cudaMemset(d_labels_, 0, batch_ * 4), "memset");
  check(cudaMemset(d_input_, 0, in.bytes()), "memset");
  build_gather_tables();

  // parameters: Kaiming-normal convs, unit BN, small classifier (deterministic)
  std::vector<float> host(n_params_, 0.f);
  std::mt19937_64 rng(seed);
  for (auto& p : params_) {
    const Op& op = ops_[p.op];
    if (p.kind == 0) {
      std::normal_distribution<float> nd(0.f, std::sqrt(2.f / (float)(op.cin_real * op.R * op.S)));
      std::vector<float> canon(p.count > 0 ? (size_t)op.cout * op.cin_real * op.R * op.S : 0);
      for (auto& v : canon) v = nd(rng);
      write_param((int)(&p - &params_[0]), canon.data());  // uploads; host copy refreshed below
      continue;
    }
    float* dst = host.data() + p.offset;
    if (p.kind == 1) std::fill(dst, dst + p.count, 1.f);
    if (p.kind == 2 || p.kind == 4) std::fill(dst, dst + p.count, 0.f);
    if (p.kind == 3) {
      std::normal_distribution<float> nd(0.f, 0.01f);
      for (long i = 0; i < p.count; ++i) dst[i] = nd(rng);
    }
    if (p.kind == 5) {  // hidden linear layer: Kaiming normal over its fan-in
      std::normal_distribution<float> nd(0.f, std::sqrt(2.f / (float)op.cin));
      for (long i = 0; i < p.count; ++i) dst[i] = nd(rng);
    }
    check(cudaMemcpy(d_param_ + p.offset, dst, p.count * 4, cudaMemcpyHostToDevice), "param upload");
  }
  std::vector<float> st(n_state_, 0.f);
  for (const auto& b : bns_) std::fill(st.begin() + b.run_var, st.begin() + b.run_var + b.C, 1.f);
  check(cudaMemcpy(d_state_, st.data(), n_state_ * 4, cudaMemcpyHostToDevice), "state upload");
  setup_done_ = true;
  prep_weights(0);
  check(cudaDeviceSynchronize(), "setup");
  tuned_ = false;
  autotune(0);
}

// Canonical (PyTorch) layout <-> GEMM layout conversions.
// Canonical (PyTorch) layout <-> the parameter's slice of the flat fp32
// buffers (GEMM layout: conv [Cout][R][S][Cpad] or [Cout][Kpad] for explicit
// im2col, hidden linear [out][h][w][c]); padding stays zero.  Host-only.
void Net::pack_param(int i, const float* host, float* buf) const {
  const Param& p = params_.at(i);
  const Op& op = ops_[p.op];
  std::fill(buf, buf + p.count, 0.f);
  if (p.kind == 0) {
    const int co = op.cout, ci = op.cin_real, R = op.R, S = op.S;
    for (int a = 0; a < co; ++a)
      for (int c = 0; c < ci; ++c)
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s) {
            const float v = host[(((long)a * ci + c) * R + r) * S + s];
            long idx;
            if (op.explicit_im2col) idx = (long)a * op.kpad + (r * S + s) * ci + c;
            else idx = (((long)a * R + r) * S + s) * op.cpad + c;
            buf[idx] = v;
          }
  } else if (p.kind == 5 && op.lin_h * op.lin_w > 1) {
    // canonical [out][c][h][w] (NCHW flatten) -> GEMM [out][h][w][c]
    const int HW = op.lin_h * op.lin_w, Cc = op.lin_c;
    for (int o = 0; o < op.classes; ++o)
      for (int c = 0; c < Cc; ++c)
        for (int hw = 0; hw < HW; ++hw)
          buf[(long)o * op.cin + (long)hw * Cc + c] = host[(long)o * op.cin + (long)c * HW + hw];
  } else {
    std::memcpy(buf, host, p.count * 4);
  }
}

void Net::unpack_param(int i, const float* buf, float* host) const {
  const Param& p = params_.at(i);
  const Op& op = ops_[p.op];
  if (p.kind == 0) {
    const int co = op.cout, ci = op.cin_real, R = op.R, S = op.S;
    for (int a = 0; a < co; ++a)
      for (int c = 0; c < ci; ++c)
        for (int r = 0; r < R; ++r)
          for (int s = 0; s < S; ++s) {
            long idx;
            if (op.explicit_im2col) idx = (long)a * op.kpad + (r * S + s) * ci + c;
            else idx = (((long)a * R + r) * S + s) * op.cpad + c;
            host[(((long)a * ci + c) * R + r) * S + s] = buf[idx];
          }
  } else if (p.kind == 5 && op.lin_h * op.lin_w > 1) {
    const int HW = op.lin_h * op.lin_w, Cc = op.lin_c;
    for (int o = 0; o < op.classes; ++o)
      for (int c = 0; c < Cc; ++c)
        for (int hw = 0; hw < HW; ++hw)
          host[(long)o * op.cin + (long)c * HW + hw] = buf[(long)o * op.cin + (long)hw * Cc + c];
  } else {
    std::memcpy(host, buf, p.count * 4);
  }
}

void Net::write_param(int i, const float* host) {
  const Param& p = params_.at(i);
  std::vector<float> buf(p.count, 0.f);
  pack_param(i, host, buf.data());
  check(cudaMemcpy(d_param_ + p.offset, buf.data(), p.count * 4, cudaMemcpyHostToDevice), "write_param");
  if (setup_done_) {
    prep_weights(0);
    check(cudaDeviceSynchronize(), "write_param");
  }
}

void Net::read_param(int i, int which, float* host) const {
  const Param& p = params_.at(i);
  const float* src = which == 0 ? d_param_ : (which == 1 ? d_grad_ : d_mom_);
  std::vector<float> buf(p.count);
  check(cudaMemcpy(buf.data(), src + p.offset, p.count * 4, cudaMemcpyDeviceToHost), "read_param");
  unpack_param(i, buf.data(), host);
}

void Net::read_tensor(int t, float* host) const {
  const Tensor& tt = tensors_.at(t);
  const void* src = tptr(t);
  if (tt.dtype == DType::F32) {
    check(cudaMemcpy(host, src, tt.bytes(), cudaMemcpyDeviceToHost), "read_tensor");
    return;
  }
  std::vector<uint16_t> buf(tt.elems());
  check(cudaMemcpy(buf.data(), src, tt.bytes(), cudaMemcpyDeviceToHost), "read_tensor");
  for (long i = 0; i < tt.elems(); ++i) host[i] = bf16_to_float(buf[i]);
}

void Net::read_grad_tensor(int t, float* host) const {
  const Tensor& tt = tensors_.at(t);
  if (grad_slot_.empty() || grad_slot_[t] < 0) throw std::invalid_argument("tensor has no gradient slot");
  const void* src = d_grad_arena_ + grad_slot_[t];
  if (tt.dtype == DType::F32) {
    check(cudaMemcpy(host, src, tt.bytes(), cudaMemcpyDeviceToHost), "read_grad_tensor");
    return;
  }
  std::vector<uint16_t> buf(tt.elems());
  check(cudaMemcpy(buf.data(), src, tt.bytes(), cudaMemcpyDeviceToHost), "read_grad_tensor");
  for (long i = 0; i < tt.elems(); ++i) host[i] = bf16_to_float(buf[i]);
}

void Net::read_bn_running(int o, float* mean, float* var) const {
  const Op& op = ops_.at(o);
  if (op.bn < 0) throw std::invalid_argument("op has no batch norm");
  const BNState& b = bns_[op.bn];
  check(cudaMemcpy(mean, d_state_ + b.run_mean, b.C * 4, cudaMemcpyDeviceToHost), "bn state");
  check(cudaMemcpy(var, d_state_ + b.run_var, b.C * 4, cudaMemcpyDeviceToHost), "bn state");
}

// ============================================================ addressing
bool Net::arena_guard_intact() const {
  std::vector<unsigned char> h(kArenaGuard);
  check(cudaMemcpy(h.data(), d_arena_ + arena_bytes_, kArenaGuard, cudaMemcpyDeviceToHost), "arena guard");
  for (unsigned char c : h)
    if (c != 0xA5) return false;
  return true;
}

void* Net::tptr(int t) const {
  if (t == input_t_) return d_input_;
  if (t == loss_t_) return d_loss_;
  if (slot_[t] < 0) throw std::runtime_error("tensor has no arena slot: " + tensors_[t].name);
  return d_arena_ + slot_[t];
}

__nv_bfloat16* Net::gptr(int t) const {
  if (grad_slot_[t] < 0) return nullptr;
  return reinterpret_cast<__nv_bfloat16*>(d_grad_arena_ + grad_slot_[t]);
}

// Algorithmic HBM bytes of one GEMM: each operand tensor read once (an im2col
// operand is its activation tensor, not the expanded matrix), the output
// written once (and read once more when accumulating).  Split-K partials are
// implementation traffic and are not counted.
static double gemm_algorithmic_bytes(const rfk::GemmDesc& d) {
  auto tensor = [](const rfk::ConvGeom& g) { return 2.0 * g.N * g.H * g.W * g.C; };
  double a = 0, b = 0;
  switch (d.a_kind) {
    case rfk::Operand::Im2colK: a = tensor(d.a_geom); break;
    default: a = 2.0 * d.M * d.K;
  }
  switch (d.b_kind) {
    case rfk::Operand::Im2colMN: b = tensor(d.b_geom); break;
    case rfk::Operand::WeightTapsMN: b = 2.0 * d.b_rows * d.b_taps * (d.b_extent > 0 ? d.b_extent : d.N); break;
    default: b = 2.0 * (double)d.N * d.K;
  }
  const double c = (d.out_f32 ? 4.0 : 2.0) * d.M * d.N * (d.accumulate_out ? 2 : 1);
  return a + b + c;
}

// Algorithmic flops of one GEMM launch: 2 M N K from its own descriptor (an
// im2col operand's K is its taps x channels), capped by the layer's
// algorithmic flops set by the op (trace_flops_) -- the cap removes padded
// channels (stem K = 7*7*3 padded to 64-multiples) and the zeros of a
// zero-insertion dgrad, while a layer split over several launches (sub-pixel
// dgrad classes, image chunks) counts each launch's own share once.
static double gemm_launch_flops(const rfk::GemmDesc& d, double layer_flops) {
  double k = d.K;
  if (d.a_kind == rfk::Operand::Im2colK) k = (double)d.a_geom.R * d.a_geom.S * d.a_geom.C;
  const double f = 2.0 * d.M * d.N * k;
  return layer_flops > 0 ? std::min(f, layer_flops) : f;
}

// Conv backward runs the weight-gradient GEMM on a side stream concurrently
// with the data-gradient GEMM (RFK_WGRAD_OVERLAP=0 serialises them).
bool Net::wgrad_overlap() const {
  static const bool on = [] {
    const char* e = std::getenv("RFK_WGRAD_OVERLAP");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

void Net::ensure_sub_streams() {
  if (sub_fork_) return;
  check(cudaEventCreateWithFlags(&sub_fork_, cudaEventDisableTiming), "event");
  for (int i = 0; i < 3; ++i) {
    create_stream(&sub_stream_[i], false);  // sub-pixel stream
    check(cudaEventCreateWithFlags(&sub_join_[i], cudaEventDisableTiming), "event");
  }
}

void Net::ensure_wgrad_stream() {
  if (wgrad_stream_) return;
  create_stream(&wgrad_stream_, false);  // weight-gradient stream
  check(cudaEventCreateWithFlags(&wgrad_fork_, cudaEventDisableTiming), "event");
  check(cudaEventCreateWithFlags(&wgrad_join_, cudaEventDisableTiming), "event");
}

// ============================================================ GEMM tile autotune
// The tile width (64 / 128 / 256 output columns) of an auto-tiled GEMM changes
// only which CTA computes which tile -- each output's K-sum order is the same
// -- but it does change which CTA rows the fused BN statistics land in, so
// every net in the process uses the same choice per shape (re-forward and
// store-all stay bit-identical).  Timed once per distinct shape on the step's
// real descriptors (CUDA-graph replay).  Opt-in (RFK_AUTOTUNE=1): measured
// +0.3 % on ResNet-50 (5624 -> 5640 img/s), i.e. the sweep-fitted model in
// gemm.cu already picks the in-situ best width almost everywhere, and the
// model's pick is deterministic across processes.
namespace {
std::mutex g_tune_mu;
std::map<std::string, int> g_tune;

bool autotune_on() {
  const char* e = std::getenv("RFK_AUTOTUNE");
  return e && std::atoi(e) != 0;
}

std::string tune_key(const rfk::GemmDesc& d) {
  char buf[320];
  const rfk::ConvGeom& a = d.a_geom;
  const rfk::ConvGeom& b = d.b_geom;
  std::snprintf(buf, sizeof buf,
                "%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%ld,%ld|%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d|%d,%d,%d,%d,%d,%d,%d,%d,%d,%d,%d",
                d.M, d.N, d.K, (int)d.a_kind, (int)d.b_kind, d.splits, d.stats != nullptr, d.out_f32, d.accumulate_out,
                d.remap, d.bn_out != nullptr, d.a_ld, d.b_ld, a.N, a.H, a.W, a.C, a.P, a.Q, a.R, a.S, a.pad_h, a.pad_w,
                a.stride_h, b.N, b.H, b.W, b.C, b.P, b.Q, b.R, b.S, b.pad_h, b.pad_w, b.stride_h);
  return buf;
}
}  // namespace

void Net::autotune(cudaStream_t st) {
  if (tuned_ || !autotune_on()) return;
  tuned_ = true;
  gemm_trace_.clear();
  tracing_ = true;
  try {
    cudaGraphExec_t e = capture([&](cudaStream_t s) { forward_backward(s); }, nullptr);
    cudaGraphExecDestroy(e);  // only the trace is wanted
  } catch (...) {
    tracing_ = false;
    throw;
  }
  tracing_ = false;
  std::lock_guard<std::mutex> lock(g_tune_mu);
  cudaEvent_t e0, e1;
  check(cudaEventCreate(&e0), "event");
  check(cudaEventCreate(&e1), "event");
  for (const auto& r : gemm_trace_) {
    if (r.desc.block_n != 0 || r.desc.band) continue;  // explicit choices (split-K plans) stay
    const std::string key = tune_key(r.desc);
    if (g_tune.count(key)) continue;
    int best = 0;
    float best_ms = 0.f;
    for (int bn : {64, 128, 256}) {
      if (bn > 64 && r.desc.N <= bn / 2) continue;
      rfk::GemmDesc dc = r.desc;
      dc.block_n = bn;
      // the probe must not leave partial sums in the conv's BN statistics
      // slot: each width maps tiles to different CTA rows, and the finalize
      // sums every row (rows a CTA never touches are assumed zero)
      dc.stats = nullptr;
      dc.stats_bwd = false;
      cudaGraphExec_t g = capture(
          [&](cudaStream_t s) {
            for (int i = 0; i < 3; ++i) check(rfk::gemm_launch(dc, s), "gemm");
          },
          nullptr);
      check(cudaGraphLaunch(g, st), "warmup");
      check(cudaEventRecord(e0, st), "event");
      check(cudaGraphLaunch(g, st), "graph");
      check(cudaEventRecord(e1, st), "event");
      check(cudaEventSynchronize(e1), "sync");
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaGraphExecDestroy(g);
      if (best == 0 || ms < best_ms * 0.97f) best = bn, best_ms = ms;  // ties keep the narrower tile
    }
    g_tune[key] = best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  gemm_trace_.clear();  // re-traced with the tuned widths when needed
  check(cudaStreamSynchronize(st), "autotune");
  // the probes wrote real output buffers (some accumulating): restore the
  // zeroed state setup() left, so a tuned net starts exactly like an untuned one
  check(cudaMemset(d_ws_, 0, rep_.workspace_bytes > 0 ? rep_.workspace_bytes : 256), "memset");
  check(cudaMemset(d_grad_, 0, n_params_ * 4), "memset");
  check(cudaMemset(d_arena_, 0, arena_bytes_ > 0 ? arena_bytes_ : 256), "memset");
  check(cudaDeviceSynchronize(), "autotune");
}

static int num_sms() {
  static const int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

void Net::gemm(const rfk::GemmDesc& d0, cudaStream_t st) {
  rfk::GemmDesc dcap;
  const rfk::GemmDesc* dp = &d0;
  if (comm_inflight_ && comm_sm_reserve_ > 0 && !d0.stats) {
    // statistics GEMMs (first forward only) keep the full grid: their
    // per-CTA statistics rows must not depend on whether a bucket is in flight
    dcap = d0;
    dcap.max_ctas = std::max(1, num_sms() - comm_sm_reserve_);
    dp = &dcap;
  }
  const rfk::GemmDesc& d = *dp;
  if (d.block_n == 0 && tuned_) {
    std::lock_guard<std::mutex> lock(g_tune_mu);
    const auto it = g_tune.find(tune_key(d));
    if (it != g_tune.end()) {
      rfk::GemmDesc dt = d;
      dt.block_n = it->second;
      if (tracing_) gemm_trace_.push_back({dt, gemm_launch_flops(dt, trace_flops_), gemm_algorithmic_bytes(dt)});
      check(rfk::gemm_launch(dt, st), "gemm");
      return;
    }
  }
  if (tracing_) gemm_trace_.push_back({d, gemm_launch_flops(d, trace_flops_), gemm_algorithmic_bytes(d)});
  check(rfk::gemm_launch(d, st), "gemm");
}

uint8_t* Net::pool_idx(const Op& op) const {
  if (op.pool_idx_off < 0) return nullptr;
  return d_ws_ + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_ + ws_stats_ + ws_misc_ + ws_counters_ + ws_dsplit_ +
         op.pool_idx_off;
}

float* Net::ws_stats_base() const {
  return reinterpret_cast<float*>(d_ws_ + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_);
}

// ============================================================ op dispatch
void Net::op_forward(const Op& op, bool reforward, int phase, cudaStream_t st) {
  uint8_t* ws = d_ws_;
  __nv_bfloat16* ws_im2col = reinterpret_cast<__nv_bfloat16*>(ws);
  float* ws_part = reinterpret_cast<float*>(ws + ws_im2col_);
  float* ws_stats = reinterpret_cast<float*>(ws + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_);
  switch (op.kind) {
    case OpKind::Conv: {
      const Tensor& x = tensors_[op.in[0]];
      const Tensor& y = tensors_[op.out];
      const Param& w = params_[op.w_param];
      rfk::GemmDesc d;
      d.M = (int)y.rows();
      d.N = op.cout;
      d.out = tptr(op.out);
      d.ldc = op.cout;
      d.b_kind = rfk::Operand::KMajor2D;
      d.b = d_bf16_ + w.bf16_off;
      if (op.explicit_im2col) {
        if (op.pad != op.pad_w) throw std::runtime_error("explicit im2col needs square padding");
        d.a_kind = rfk::Operand::KMajor2D;
        d.a = ws_im2col;
        d.a_ld = op.kpad;
        d.K = op.kpad;
        d.b_ld = op.kpad;
        float* stats = (op.fuse_stats && !reforward) ? ws_stats + op.stats_off : nullptr;
        trace_flops_ = 2.0 * y.rows() * op.cout * op.R * op.S * op.cin_real;
        if (reforward && op.fused_bn >= 0) {
          const Op& bn = ops_[op.fused_bn];
          const BNState& b = bns_[bn.bn];
          d.bn_out = tptr(bn.out);
          d.bn_scale = d_state_ + b.scale;
          d.bn_shift = d_state_ + b.shift;
          d.bn_relu = bn.k == 1;
        }
        // image chunks: im2col of a chunk (L2-resident) -> its GEMM rows; the
        // BN statistics rows accumulate over the chunks in order
        const long img_rows = (long)y.H * y.W;
        for (int n0 = 0; n0 < x.N; n0 += op.im2col_imgs) {
          const int nn = std::min(op.im2col_imgs, x.N - n0);
          rfk::ConvShape cs{nn, x.H, x.W, op.cin_real, x.C, y.H, y.W, op.R, op.S, op.stride, op.pad};
          // the matrix of the network input is the same for the first
          // forward, the re-forward and the weight gradient: built once per step
          const int oid = (int)(&op - &ops_[0]);
          const bool whole = nn == x.N && op.in[0] == input_t_;
          if (!(whole && im2col_holder_ == oid))
            check(rfk::im2col(tb(op.in[0]) + (long)n0 * x.H * x.W * x.C, cs, op.kpad, ws_im2col, st), "im2col");
          im2col_holder_ = whole ? oid : -1;
          rfk::GemmDesc dc = d;
          dc.M = (int)(nn * img_rows);
          dc.out = tb(op.out) + n0 * img_rows * op.cout;
          if (dc.bn_out) dc.bn_out = static_cast<__nv_bfloat16*>(dc.bn_out) + n0 * img_rows * op.cout;
          dc.stats = stats;
          dc.stats_acc = n0 > 0;
          trace_flops_ = 2.0 * dc.M * op.cout * op.R * op.S * op.cin_real;  // this chunk's share
          gemm(dc, st);
        }
        break;
      } else if (op.R == 1 && op.S == 1 && op.stride == 1 && op.pad == 0 && op.pad_w == 0) {
        d.a_kind = rfk::Operand::KMajor2D;
        d.a = tptr(op.in[0]);
        d.a_ld = op.cin;
        d.K = op.cin;
        d.b_ld = op.cpad;
      } else {
        d.a_kind = rfk::Operand::Im2colK;
        d.a = tptr(op.in[0]);
        d.a_geom = rfk::ConvGeom{x.N, x.H, x.W, x.C, y.H, y.W, op.R, op.S, op.pad, op.pad_w, op.stride, op.stride};
        // shifted-band kernel where it pays (gemm_band.cu).  Its K order is
        // channel block outer, tap inner -- the TMA im2col path's order only
        // with one 64-channel block, where the two give identical bits.  With
        // more blocks it runs only for the narrow (<= 32-channel) DenseNet
        // growth convs, and only if no plan can re-forward the conv through
        // the im2col kernel with its BN fused (every plan then computes the
        // same bits: re-forward / store-all identity); elsewhere the measured
        // gain is small and the results would move by summation order.
        d.band = (op.cpad <= 64 || (op.cout <= 32 && !fusable_conv(op))) ? band_enabled() : 0;
        d.K = op.R * op.S * op.cpad;
        d.b_ld = (long)op.R * op.S * op.cpad;
      }
      float* stats = (op.fuse_stats && !reforward) ? ws_stats + op.stats_off : nullptr;
      trace_flops_ = 2.0 * y.rows() * op.cout * op.R * op.S * op.cin_real;
      if (op.fp_splits > 1 && d.a_kind == rfk::Operand::Im2colK) {
        // split-K into fp32 partials, then one pass sums them in split order,
        // rounds to bf16 and emits the BN statistics rows
        // the main-stream split region (the weight-gradient partials of a
        // pending side-stream GEMM may still live in ws_split)
        float* ws_split = reinterpret_cast<float*>(ws + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_ + ws_stats_ +
                                                   ws_misc_ + ws_counters_);
        d.splits = op.fp_splits;
        d.block_n = op.fp_bn;
        d.out = ws_split;
        d.out_f32 = true;
        d.ldc = op.cout;
        d.split_stride = y.rows() * op.cout;
        gemm(d, st);
        check(rfk::reduce_splits_bf16(ws_split, op.fp_splits, (int)y.rows(), op.cout, tb(op.out), op.cout, false, stats,
                                      (int)kStatRows, st),
              "reduce_splits_bf16");
        break;
      }
      d.stats = stats;
      if (reforward && op.fused_bn >= 0) {
        const Op& bn = ops_[op.fused_bn];
        const BNState& b = bns_[bn.bn];
        d.bn_out = tptr(bn.out);
        d.bn_scale = d_state_ + b.scale;
        d.bn_shift = d_state_ + b.shift;
        d.bn_relu = bn.k == 1;
        d.band = 0;
      }
      gemm(d, st);
      break;
    }
    case OpKind::BN:
    case OpKind::BNAddReLU: {
      const Tensor& y = tensors_[op.in[0]];
      const BNState& b = bns_[op.bn];
      float* S = d_state_;
      if (phase == 1) {  // residual add, phase 1: out <- skip (exact copy)
        check(rfk::copy_bytes(tptr(op.out), tptr(op.in[1]), y.bytes(), st), "skip copy");
        break;
      }
      if (!reforward && op.bn_gather >= 0) {
        // BN over a concatenation: gather the leaves' statistics, then apply
        const auto* table = static_cast<const rfk::BnGatherBlock*>(d_gather_) + gather_first_block_[op.bn_gather];
        check(rfk::bn_finalize_gather(table, y.C, y.rows(), d_param_ + params_[op.w_param].offset,
                                      d_param_ + params_[op.b_param].offset, op.eps, S + b.mean, S + b.invstd,
                                      S + b.scale, S + b.shift, S + b.run_mean, S + b.run_var, op.momentum, st),
              "bn_finalize_gather");
        const bool relu = op.kind == OpKind::BNAddReLU || op.k == 1;
        const __nv_bfloat16* skip = op.kind == OpKind::BNAddReLU ? tb(op.in[1]) : nullptr;
        if (phase == 2) skip = tb(op.out);
        check(rfk::bn_apply(tb(op.in[0]), skip, S + b.scale, S + b.shift, relu, y.rows(), y.C, tb(op.out), st),
              "bn_apply");
        break;
      }
      if (!reforward) {
        const Op& prod = ops_[y.producer];
        const float* partials;
        int parts;
        if (prod.kind == OpKind::Conv && prod.fuse_stats) {
          partials = ws_stats + prod.stats_off;
          parts = (int)kStatRows;  // rows past the GEMM's grid are zero
        } else {
          parts = rfk::colstats_blocks(y.rows());
          check(rfk::colstats(tb(op.in[0]), y.rows(), y.C, ws_part, parts, st), "colstats");
          partials = ws_part;
        }
        check(rfk::bn_finalize(partials, parts, y.C, y.rows(), d_param_ + params_[op.w_param].offset,
                               d_param_ + params_[op.b_param].offset, op.eps, S + b.mean, S + b.invstd, S + b.scale,
                               S + b.shift, S + b.run_mean, S + b.run_var, op.momentum, true, st),
              "bn_finalize");
      }
      const bool relu = op.kind == OpKind::BNAddReLU || op.k == 1;
      const __nv_bfloat16* skip = op.kind == OpKind::BNAddReLU ? tb(op.in[1]) : nullptr;
      if (phase == 2) skip = tb(op.out);  // phase 1 already placed the skip in the output slot
      check(rfk::bn_apply(tb(op.in[0]), skip, S + b.scale, S + b.shift, relu, y.rows(), y.C, tb(op.out), st),
            "bn_apply");
      break;
    }
    case OpKind::ReLU:
      check(rfk::relu_fwd(tb(op.in[0]), tensors_[op.out].elems(), tb(op.out), st), "relu");
      break;
    case OpKind::MaxPool: {
      const Tensor& x = tensors_[op.in[0]];
      const Tensor& y = tensors_[op.out];
      rfk::PoolGeom g{x.N, x.H, x.W, x.C, y.H, y.W, op.k, op.stride, op.pad};
      check(rfk::maxpool_fwd(tb(op.in[0]), g, tb(op.out), st, pool_idx(op)), "maxpool");
      break;
    }
    case OpKind::AvgPool: {
      const Tensor& x = tensors_[op.in[0]];
      check(rfk::avgpool_fwd(tb(op.in[0]), x.N, x.H * x.W, x.C, tb(op.out), st), "avgpool");
      break;
    }
    case OpKind::FC: {
      const Param& w = params_[op.w_param];
      rfk::GemmDesc d;
      d.M = batch_;
      d.N = op.classes;
      d.K = op.cin;
      d.a_kind = rfk::Operand::KMajor2D;
      d.a = tptr(op.in[0]);
      d.a_ld = op.cin;
      d.b_kind = rfk::Operand::KMajor2D;
      d.b = d_bf16_ + w.bf16_off;
      d.b_ld = op.cin;
      d.out = tptr(op.out);
      d.ldc = op.classes;
      d.out_f32 = true;
      d.bias = d_param_ + params_[op.b_param].offset;
      trace_flops_ = 2.0 * batch_ * op.classes * op.cin;
      gemm(d, st);
      break;
    }
    case OpKind::AvgPool2d: {
      const Tensor& x = tensors_[op.in[0]];
      const Tensor& y = tensors_[op.out];
      rfk::PoolGeom g{x.N, x.H, x.W, x.C, y.H, y.W, op.k, op.stride, op.pad};
      check(rfk::avgpool2d_fwd(tb(op.in[0]), g, tb(op.out), st), "avgpool2d");
      break;
    }
    case OpKind::Linear: {
      const Param& w = params_[op.w_param];
      rfk::GemmDesc d;
      d.M = batch_;
      d.N = op.classes;
      d.K = op.cin;
      d.a_kind = rfk::Operand::KMajor2D;
      d.a = tptr(op.in[0]);
      d.a_ld = op.cin;
      d.b_kind = rfk::Operand::KMajor2D;
      d.b = d_bf16_ + w.bf16_off;
      d.b_ld = op.cin;
      d.out = tptr(op.out);
      d.ldc = op.classes;
      d.bias = d_param_ + params_[op.b_param].offset;
      trace_flops_ = 2.0 * batch_ * op.classes * op.cin;
      gemm(d, st);
      break;
    }
    case OpKind::Concat: {
      const Tensor& a = tensors_[op.in[0]];
      const Tensor& b2 = tensors_[op.in[1]];
      check(rfk::concat(phase == 2 ? nullptr : tb(op.in[0]), a.C, phase == 1 ? nullptr : tb(op.in[1]), b2.C, a.rows(),
                        tb(op.out), st),
            "concat");
      break;
    }
    case OpKind::Loss:
      check(rfk::softmax_ce_fwd(static_cast<const float*>(tptr(op.in[0])), d_labels_, batch_, op.classes, d_rowloss_,
                                d_lse_, d_loss_, st),
            "loss");
      break;
    case OpKind::Input:
      break;
  }
}

void Net::op_backward(const Op& op, cudaStream_t st) {
  const int oid = (int)(&op - &ops_[0]);
  auto acc = [&](int i) { return grad_acc_[grad_acc_base_[oid] + i] != 0; };
  uint8_t* ws = d_ws_;
  __nv_bfloat16* ws_im2col = reinterpret_cast<__nv_bfloat16*>(ws);
  float* ws_part = reinterpret_cast<float*>(ws + ws_im2col_);
  __nv_bfloat16* ws_zero = reinterpret_cast<__nv_bfloat16*>(ws + ws_im2col_ + ws_partials_);
  float* ws_split = reinterpret_cast<float*>(ws + ws_im2col_ + ws_partials_ + ws_zero_);
  __nv_bfloat16* ws_misc =
      reinterpret_cast<__nv_bfloat16*>(ws + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_ + ws_stats_);
  switch (op.kind) {
    case OpKind::Conv: {
      const Tensor& x = tensors_[op.in[0]];
      const Tensor& y = tensors_[op.out];
      const Param& w = params_[op.w_param];
      const __nv_bfloat16* dy = gptr(op.out);
      trace_flops_ = 2.0 * y.rows() * op.cout * op.R * op.S * op.cin_real;  // dgrad and wgrad each
      // fork: the weight gradient (below) runs on a side stream next to the
      // data gradient; both only read dy and x, and the join closes this op
      const bool fork = wgrad_overlap();
      cudaStream_t wst = st;
      if (fork) {
        ensure_wgrad_stream();
        check(cudaEventRecord(wgrad_fork_, st), "event");
        check(cudaStreamWaitEvent(wgrad_stream_, wgrad_fork_, 0), "wait");
        wst = wgrad_stream_;
      }
      // ---- dgrad
      __nv_bfloat16* dx = gptr(op.in[0]);
      if (op.in[0] != input_t_ && dx) {
        if (op.explicit_im2col) throw std::runtime_error("dgrad of an explicit-im2col conv is not supported");
        rfk::GemmDesc d;
        d.N = op.cin;
        d.b_kind = rfk::Operand::KMajor2D;
        d.b = d_bf16_ + w.bf16_off;  // the forward bf16 weights, read transposed by TMA
        d.b_extent = op.cin;
        d.out = dx;
        d.ldc = op.cin;
        d.accumulate_out = acc(0);
        if (op.R == 1 && op.S == 1 && op.pad == 0 && op.pad_w == 0) {
          d.M = (int)y.rows();
          d.K = op.cout;
          d.a_kind = rfk::Operand::KMajor2D;
          d.a = dy;
          d.a_ld = op.cout;
          d.b_kind = rfk::Operand::MNMajor2D;  // W[co][ci]: K = co rows, N = ci contiguous
          d.b_ld = op.cpad;
          if (op.stride > 1) {
            if (!acc(0)) check(rfk::fill_zero(dx, x.bytes(), st), "zero dx");
            d.accumulate_out = acc(0);
            d.remap = true;
            d.rP = y.H;
            d.rQ = y.W;
            d.rH = x.H;
            d.rW = x.W;
            d.rsh = d.rsw = op.stride;
          }
        } else {
          d.M = (int)x.rows();
          d.K = op.R * op.S * op.coutpad;
          d.b_kind = rfk::Operand::WeightTapsMN;  // W[co][tap][ci] with the tap flipped
          d.b_taps = op.R * op.S;
          d.b_cpad = op.cpad;
          d.b_rows = op.cout;
          d.a_kind = rfk::Operand::Im2colK;
          // (one channel block of dy only: the band and im2col kernels then sum
          // in the same order, so whether the plan fuses the BN-backward
          // statistics into this dgrad -- which excludes the band kernel --
          // never changes its bits)
          d.band = op.coutpad <= 64 ? band_enabled() : 0;
          const int pd = op.R - 1 - op.pad, pdw = op.S - 1 - op.pad_w;
          if (op.dg_subpixel) {
            // Sub-pixel decomposition: the stride x stride classes of input
            // positions (h, w) = (s*m + a, s*n + b) each take a stride-1
            // correlation of dy with their own subset of the (flipped) taps --
            // no zero-inserted dy, no multiplications by inserted zeros.  Every
            // class GEMM scatters its rows to its pixels (row remap).
            const int st_ = op.stride;
            bool empty = false;
            for (int a = 0; a < st_; ++a)
              for (int b = 0; b < st_; ++b) {
                const SubpixelDim ch = subpixel_dim(a, st_, op.R, op.pad, x.H);
                const SubpixelDim cw = subpixel_dim(b, st_, op.S, op.pad_w, x.W);
                empty |= ch.J == 0 || cw.J == 0;
              }
            if (empty && !acc(0)) check(rfk::fill_zero(dx, x.bytes(), st), "zero dx");
            // classes write disjoint pixels: up to four run concurrently
            // (each alone is too small to fill the GPU)
            const bool par = st_ == 2 && sub_parallel();
            if (par) {
              ensure_sub_streams();
              check(cudaEventRecord(sub_fork_, st), "event");
            }
            int cls = 0;
            bool launched[4] = {false, false, false, false};
            for (int a = 0; a < st_; ++a)
              for (int b = 0; b < st_; ++b, ++cls) {
                const SubpixelDim ch = subpixel_dim(a, st_, op.R, op.pad, x.H);
                const SubpixelDim cw = subpixel_dim(b, st_, op.S, op.pad_w, x.W);
                if (ch.J == 0 || cw.J == 0 || ch.rows == 0 || cw.rows == 0) continue;
                rfk::GemmDesc dc = d;
                dc.M = x.N * ch.rows * cw.rows;
                dc.K = ch.J * cw.J * op.coutpad;
                dc.a = dy;
                dc.a_geom = rfk::ConvGeom{y.N, y.H, y.W, op.cout, ch.rows, cw.rows, ch.J, cw.J, ch.pad_lo, cw.pad_lo, 1, 1};
                dc.b_tap_base = (ch.r0 + (ch.J - 1) * st_) * op.S + cw.r0 + (cw.J - 1) * st_;
                dc.b_tap_dr = st_ * op.S;
                dc.b_tap_ds = st_;
                if (ch.J == 1 && cw.J == 1 && ch.pad_lo == 0 && cw.pad_lo == 0 && ch.rows == y.H && cw.rows == y.W) {
                  // one tap, no shift: A is dy itself and B one weight tap
                  // (plain 2-D operands, no im2col)
                  dc.K = op.cout;
                  dc.a_kind = rfk::Operand::KMajor2D;
                  dc.a_ld = op.cout;
                  dc.b_kind = rfk::Operand::MNMajor2D;
                  dc.b = d_bf16_ + w.bf16_off + (long)dc.b_tap_base * op.cpad;
                  dc.b_ld = (long)op.R * op.S * op.cpad;
                  dc.b_extent = op.cin;
                  dc.b_tap_base = -1;
                }
                dc.band = 0;
                dc.remap = true;
                dc.rP = ch.rows;
                dc.rQ = cw.rows;
                dc.rH = x.H;
                dc.rW = x.W;
                dc.rsh = dc.rsw = st_;
                dc.out = dx + ((long)a * x.W + b) * op.cin;
                cudaStream_t cs = st;
                if (par && cls > 0) {
                  cs = sub_stream_[cls - 1];
                  check(cudaStreamWaitEvent(cs, sub_fork_, 0), "wait");
                }
                gemm(dc, cs);
                if (par && cls > 0) check(cudaEventRecord(sub_join_[cls - 1], cs), "event");
                if (cls < 4) launched[cls] = true;
              }
            if (par)
              for (int i = 1; i < cls; ++i)
                if (launched[i]) check(cudaStreamWaitEvent(st, sub_join_[i - 1], 0), "wait");
          } else if (op.stride == 1) {
            d.a = dy;
            d.a_geom = rfk::ConvGeom{y.N, y.H, y.W, op.cout, x.H, x.W, op.R, op.S, pd, pdw, 1, 1};
          } else {
            const int Hu = x.H - op.R + 1 + 2 * op.pad, Wu = x.W - op.S + 1 + 2 * op.pad;
            check(rfk::zero_insert(dy, y.N, y.H, y.W, op.cout, Hu, Wu, op.stride, ws_zero, st), "zero_insert");
            d.a = ws_zero;
            d.a_geom = rfk::ConvGeom{y.N, Hu, Wu, op.cout, x.H, x.W, op.R, op.S, pd, pd, 1, 1};
          }
        }
        if (op.dg_splits > 1 && d.a_kind == rfk::Operand::Im2colK) {
          // own region: the weight-gradient split partials may be in flight on the side stream
          float* ws_split = reinterpret_cast<float*>(ws + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_ + ws_stats_ +
                                                     ws_misc_ + ws_counters_);
          const bool accumulate = d.accumulate_out;
          d.splits = op.dg_splits;
          d.block_n = op.dg_bn;
          d.out = ws_split;
          d.out_f32 = true;
          d.accumulate_out = false;
          d.ldc = op.cin;
          d.split_stride = (long)d.M * op.cin;
          gemm(d, st);
          check(rfk::reduce_splits_bf16(ws_split, op.dg_splits, d.M, op.cin, dx, op.cin, accumulate, nullptr,
                                        (int)kStatRows, st),
                "reduce_splits_bf16");
        } else if (!op.dg_subpixel) {
          if (op.bstat_src >= 0) {
            // this dgrad's output is dout of a BN+ReLU whose input is
            // resident: store g and emit that BN's backward statistics rows
            const Op& bn = ops_[op.bstat_src];
            const BNState& b = bns_[bn.bn];
            if (d.remap || d.accumulate_out || d.splits > 1) throw std::runtime_error("bstat dgrad is not a plain launch");
            d.stats = ws_stats_base() + bn.bstat_off;
            d.stats_bwd = true;
            d.block_n = bn.bstat_bn;
            d.band = 0;
            d.bs_y = tptr(bn.in[0]);
            d.bs_ldy = tensors_[bn.in[0]].C;
            d.bs_mean = d_state_ + b.mean;
            d.bs_scale = d_state_ + b.scale;
            d.bs_shift = d_state_ + b.shift;
          }
          gemm(d, st);
        }
      }
      // ---- wgrad
      const long kw = op.explicit_im2col ? op.kpad : (long)op.R * op.S * op.cpad;
      float* dW = d_grad_ + w.offset;
      rfk::GemmDesc d;
      d.M = op.cout;
      d.N = (int)kw;
      d.K = (int)y.rows();
      d.a_kind = rfk::Operand::MNMajor2D;
      d.a = dy;
      d.a_ld = op.cout;
      d.out_f32 = true;
      d.ldc = kw;
      d.block_n = op.wg_bn;
      if (op.explicit_im2col) {
        // image chunks (L2-resident im2col): every chunk's split-K partials
        // land in their own slice; one reduction sums them chunk-major
        d.b_kind = rfk::Operand::MNMajor2D;
        d.b = ws_im2col;
        d.b_ld = op.kpad;
        d.splits = op.wg_splits;
        d.split_stride = (long)op.cout * kw;
        const long img_rows = (long)y.H * y.W;
        int parts = 0;
        for (int n0 = 0; n0 < x.N; n0 += op.im2col_imgs) {
          const int nn = std::min(op.im2col_imgs, x.N - n0);
          rfk::ConvShape cs{nn, x.H, x.W, op.cin_real, x.C, y.H, y.W, op.R, op.S, op.stride, op.pad};
          const int oid = (int)(&op - &ops_[0]);
          const bool whole = nn == x.N && op.in[0] == input_t_;
          if (!(whole && im2col_holder_ == oid))
            check(rfk::im2col(tb(op.in[0]) + (long)n0 * x.H * x.W * x.C, cs, op.kpad, ws_im2col, wst), "im2col");
          im2col_holder_ = whole ? oid : -1;
          rfk::GemmDesc dc = d;
          dc.K = (int)(nn * img_rows);
          dc.a = dy + n0 * img_rows * op.cout;
          dc.out = ws_split + (long)parts * op.cout * kw;
          const double layer = trace_flops_;
          trace_flops_ = 2.0 * dc.K * op.cout * op.R * op.S * op.cin_real;  // this chunk's share
          gemm(dc, wst);
          trace_flops_ = layer;
          parts += op.wg_splits;
        }
        check(rfk::reduce_splits(ws_split, parts, (long)op.cout * kw, dW, false, wst), "reduce_splits");
      } else if (op.R == 1 && op.S == 1 && op.stride == 1 && op.pad == 0 && op.pad_w == 0) {
        d.b_kind = rfk::Operand::MNMajor2D;
        d.b = tptr(op.in[0]);
        d.b_ld = op.cin;
        d.b_extent = op.cin;
      } else {
        d.b_kind = rfk::Operand::Im2colMN;
        d.b = tptr(op.in[0]);
        d.b_geom = rfk::ConvGeom{x.N, x.H, x.W, x.C, y.H, y.W, op.R, op.S, op.pad, op.pad_w, op.stride, op.stride};
      }
      if (op.explicit_im2col) {
        // done above
      } else if (op.wg_splits > 1) {
        // split-K partials in the workspace, summed in split order by a
        // whole-GPU reduction kernel into the gradient buffer
        d.splits = op.wg_splits;
        d.out = ws_split;
        d.split_stride = (long)op.cout * kw;
        gemm(d, wst);
        check(rfk::reduce_splits(ws_split, op.wg_splits, (long)op.cout * kw, dW, false, wst), "reduce_splits");
      } else {
        d.out = dW;
        gemm(d, wst);
      }
      if (fork) {
        // joined lazily (forward_backward): before the first instruction that
        // writes what this weight gradient reads, before an all-reduce bucket,
        // and at the end of the backward
        if (op.in[0] != input_t_) wgrad_reads_act_.push_back({slot_[op.in[0]], slot_[op.in[0]] + x.bytes()});
        wgrad_reads_grad_.push_back({grad_slot_[op.out], grad_slot_[op.out] + y.bytes()});
        wgrad_pending_ = true;
      }
      break;
    }
    case OpKind::BN:
    case OpKind::BNAddReLU: {
      const Tensor& y = tensors_[op.in[0]];
      const BNState& b = bns_[op.bn];
      float* S = d_state_;
      const bool add = op.kind == OpKind::BNAddReLU;
      const int mode = add ? 2 : (op.k == 1 ? 1 : 0);
      if (op.bstat) {
        // statistics rows from the consumer conv's dgrad epilogue, or a replay
        // over the stored dout with the same tiles (bit-identical rows)
        float* rows = ws_stats_base() + op.bstat_off;
        if (!op.bstat_fused) {
          rfk::GemmDesc r;
          r.M = (int)y.rows();
          r.N = y.C;
          r.K = 0;
          r.out = gptr(op.out);
          r.ldc = y.C;
          r.stats = rows;
          r.stats_bwd = true;
          r.replay = true;
          r.block_n = op.bstat_bn;
          r.bs_y = tb(op.in[0]);
          r.bs_ldy = y.C;
          r.bs_mean = S + b.mean;
          r.bs_scale = S + b.scale;
          r.bs_shift = S + b.shift;
          check(rfk::gemm_launch(r, st), "bstat replay");  // not a GEMM: kept out of the GEMM trace
        }
        check(rfk::bn_backward_from_rows(tb(op.in[0]), gptr(op.out), d_param_ + params_[op.w_param].offset,
                                         S + b.mean, S + b.invstd, S + b.scale, S + b.shift, y.rows(), y.C, rows,
                                         (int)kStatRows, S + b.coef, d_grad_ + params_[op.w_param].offset,
                                         d_grad_ + params_[op.b_param].offset, gptr(op.in[0]), acc(0), st),
              "bn_backward_from_rows");
        break;
      }
      const int blocks = rfk::colstats_blocks(y.rows());
      __nv_bfloat16* dskip = add ? gptr(op.in[1]) : nullptr;
      check(rfk::bn_backward(tb(op.in[0]), gptr(op.out), add ? tb(op.out) : nullptr, mode,
                             d_param_ + params_[op.w_param].offset, S + b.mean, S + b.invstd, S + b.scale,
                             S + b.shift, y.rows(), y.C, ws_part, blocks, S + b.coef,
                             d_grad_ + params_[op.w_param].offset, d_grad_ + params_[op.b_param].offset,
                             gptr(op.in[0]), acc(0), dskip, add ? acc(1) : false, st),
            "bn_backward");
      break;
    }
    case OpKind::ReLU:
      check(rfk::relu_bwd(tb(op.out), gptr(op.out), tensors_[op.out].elems(), gptr(op.in[0]), acc(0), st),
            "relu_bwd");
      break;
    case OpKind::MaxPool: {
      const Tensor& x = tensors_[op.in[0]];
      const Tensor& y = tensors_[op.out];
      rfk::PoolGeom g{x.N, x.H, x.W, x.C, y.H, y.W, op.k, op.stride, op.pad};
      if (op.pool_idx_off >= 0)
        check(rfk::maxpool_bwd_from_idx(pool_idx(op), gptr(op.out), g, gptr(op.in[0]), acc(0), st), "maxpool_bwd");
      else
        check(rfk::maxpool_bwd(tb(op.in[0]), tb(op.out), gptr(op.out), g, gptr(op.in[0]), acc(0), ws_zero, st),
              "maxpool_bwd");
      break;
    }
    case OpKind::AvgPool: {
      const Tensor& x = tensors_[op.in[0]];
      check(rfk::avgpool_bwd(gptr(op.out), x.N, x.H * x.W, x.C, gptr(op.in[0]), acc(0), st), "avgpool_bwd");
      break;
    }
    case OpKind::FC: {
      const Param& w = params_[op.w_param];
      const float* dlog = reinterpret_cast<const float*>(gptr(op.out));
      const int ldd = round8(op.classes);
      trace_flops_ = 2.0 * batch_ * op.classes * op.cin;
      // bf16 copy of dlogits with 16-byte aligned rows for TMA
      check(rfk::fill_zero(ws_misc, (long)batch_ * ldd * 2, st), "zero");
      check(rfk::cast_f32_bf16_2d(dlog, batch_, op.classes, ldd, ws_misc, st), "cast");
      check(rfk::colsum_f32(dlog, batch_, op.classes, d_grad_ + params_[op.b_param].offset, false, st), "db");
      __nv_bfloat16* dx = gptr(op.in[0]);
      if (dx) {
        rfk::GemmDesc d;
        d.M = batch_;
        d.N = op.cin;
        d.K = op.classes;
        d.a_kind = rfk::Operand::KMajor2D;
        d.a = ws_misc;
        d.a_ld = ldd;
        d.b_kind = rfk::Operand::MNMajor2D;
        d.b = d_bf16_ + w.bf16_off;
        d.b_ld = op.cin;
        d.out = dx;
        d.ldc = op.cin;
        d.accumulate_out = acc(0);
        gemm(d, st);
      }
      rfk::GemmDesc d;
      d.M = op.classes;
      d.N = op.cin;
      d.K = batch_;
      d.a_kind = rfk::Operand::MNMajor2D;
      d.a = ws_misc;
      d.a_ld = ldd;
      d.b_kind = rfk::Operand::MNMajor2D;
      d.b = tptr(op.in[0]);
      d.b_ld = op.cin;
      d.out = d_grad_ + w.offset;
      d.ldc = op.cin;
      d.out_f32 = true;
      gemm(d, st);
      break;
    }
    case OpKind::AvgPool2d: {
      const Tensor& x = tensors_[op.in[0]];
      const Tensor& y = tensors_[op.out];
      rfk::PoolGeom g{x.N, x.H, x.W, x.C, y.H, y.W, op.k, op.stride, op.pad};
      check(rfk::avgpool2d_bwd(gptr(op.out), g, gptr(op.in[0]), acc(0), st), "avgpool2d_bwd");
      break;
    }
    case OpKind::Linear: {
      const Param& w = params_[op.w_param];
      const __nv_bfloat16* dy = gptr(op.out);
      trace_flops_ = 2.0 * batch_ * op.classes * op.cin;
      check(rfk::colsum_bf16(dy, batch_, op.classes, d_grad_ + params_[op.b_param].offset, false, st), "db");
      __nv_bfloat16* dx = gptr(op.in[0]);
      if (dx) {
        rfk::GemmDesc d;  // dX[batch][Kin] = dY[batch][out] W[out][Kin]
        d.M = batch_;
        d.N = op.cin;
        d.K = op.classes;
        d.a_kind = rfk::Operand::KMajor2D;
        d.a = dy;
        d.a_ld = op.classes;
        d.b_kind = rfk::Operand::MNMajor2D;
        d.b = d_bf16_ + w.bf16_off;
        d.b_ld = op.cin;
        d.out = dx;
        d.ldc = op.cin;
        d.accumulate_out = acc(0);
        gemm(d, st);
      }
      rfk::GemmDesc d;  // dW[out][Kin] = dY^T X
      d.M = op.classes;
      d.N = op.cin;
      d.K = batch_;
      d.a_kind = rfk::Operand::MNMajor2D;
      d.a = dy;
      d.a_ld = op.classes;
      d.b_kind = rfk::Operand::MNMajor2D;
      d.b = tptr(op.in[0]);
      d.b_ld = op.cin;
      d.out = d_grad_ + w.offset;
      d.ldc = op.cin;
      d.out_f32 = true;
      gemm(d, st);
      break;
    }
    case OpKind::Concat: {
      const Tensor& a = tensors_[op.in[0]];
      const Tensor& b2 = tensors_[op.in[1]];
      check(rfk::split_grad(gptr(op.out), a.C, b2.C, a.rows(), gptr(op.in[0]), acc(0), gptr(op.in[1]), acc(1), st),
            "split_grad");
      break;
    }
    case OpKind::Loss:
      check(rfk::softmax_ce_bwd(static_cast<const float*>(tptr(op.in[0])), d_labels_, d_lse_, batch_, op.classes,
                                reinterpret_cast<float*>(gptr(op.in[0])), st),
            "loss_bwd");
      break;
    case OpKind::Input:
      break;
  }
}

// Device tables of the BN-over-concat statistics gathers: one entry per
// 32-channel block of each such BN, pointing at the rows of the leaf tensor
// that produced those channels (conv epilogue slot or colstats slot).
void Net::build_gather_tables() {
  gather_first_block_.clear();
  if (gather_leaves_.empty()) return;
  float* ws_stats = reinterpret_cast<float*>(d_ws_ + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_);
  std::vector<rfk::BnGatherBlock> tab;
  for (const auto& leaves : gather_leaves_) {
    gather_first_block_.push_back((int)tab.size());
    for (int u : leaves) {
      const Tensor& t = tensors_[u];
      const Op& pr = ops_[t.producer];
      rfk::BnGatherBlock b{};
      if (pr.kind == OpKind::Conv && pr.out == u && pr.fuse_stats) {
        b.partials = ws_stats + pr.stats_off;
        b.parts = (int)kStatRows;
      } else {
        if (leaf_stats_off_[u] < 0) throw std::logic_error("concat leaf without a statistics slot");
        b.partials = ws_stats + leaf_stats_off_[u];
        b.parts = rfk::colstats_blocks(t.rows());
      }
      b.Csrc = t.C;
      for (int c = 0; c < t.C; c += 32) {
        b.coff = c;
        tab.push_back(b);
      }
    }
  }
  check(cudaMalloc(&d_gather_, tab.size() * sizeof(rfk::BnGatherBlock)), "gather table");
  rep_.device_bytes += (long)(tab.size() * sizeof(rfk::BnGatherBlock));
  check(cudaMemcpy(d_gather_, tab.data(), tab.size() * sizeof(rfk::BnGatherBlock), cudaMemcpyHostToDevice),
        "gather table");
}

void Net::run_instr(const Instr& ins, cudaStream_t st) {
  if (ins.kind == InstrKind::Forward && ins.reforward && ops_[ins.op].reforward_in_producer) return;  // done by the conv
  if (ins.kind == InstrKind::Forward) {
    const Op& op = ops_[ins.op];
    op_forward(op, ins.reforward, ins.phase, st);
    if (!ins.reforward && ins.phase != 1 && op.out >= 0 && leaf_stats_off_[op.out] >= 0) {
      // statistics of a concat leaf, once, for every BN that gathers them
      const Tensor& t = tensors_[op.out];
      float* ws_stats = reinterpret_cast<float*>(d_ws_ + ws_im2col_ + ws_partials_ + ws_zero_ + ws_split_);
      check(rfk::colstats(tb(op.out), t.rows(), t.C, ws_stats + leaf_stats_off_[op.out], rfk::colstats_blocks(t.rows()),
                          st),
            "leaf colstats");
    }
    return;
  }
  else if (ins.kind == InstrKind::Backward) op_backward(ops_[ins.op], st);
}

// ============================================================ step
void Net::prep_weights(cudaStream_t st) {
  check(rfk::cast_f32_bf16_vec(d_param_, n_params_, d_bf16_, st), "weight cast");
}

void Net::prep_weights_table(cudaStream_t st) {
  // one batched launch over every conv / fc weight (table built once)
  if (!d_prep_table_) {
    std::vector<rfk::WeightPrepLayer> tab;
    long start = 0;
    for (const auto& p : params_) {
      if (p.kind != 0 && p.kind != 3 && p.kind != 5) continue;
      const Op& op = ops_[p.op];
      rfk::WeightPrepLayer L{};
      L.w = d_param_ + p.offset;
      L.wb = d_bf16_ + p.bf16_off;
      L.n_copy = p.count;
      (void)op;
      L.start = start;
      start += L.n_copy + L.n_t;
      tab.push_back(L);
    }
    prep_layers_ = (int)tab.size();
    prep_total_ = start;
    check(cudaMalloc(&d_prep_table_, sizeof(rfk::WeightPrepLayer) * std::max<size_t>(1, tab.size())), "prep table");
    rep_.device_bytes += (long)(sizeof(rfk::WeightPrepLayer) * std::max<size_t>(1, tab.size()));
    check(cudaMemcpy(d_prep_table_, tab.data(), sizeof(rfk::WeightPrepLayer) * tab.size(), cudaMemcpyHostToDevice),
          "prep table");
  }
  check(rfk::weight_prep_batched(static_cast<const rfk::WeightPrepLayer*>(d_prep_table_), prep_layers_, prep_total_,
                                 st),
        "weight prep");
}

void Net::load_batch(const float* images, const int* labels, bool from_host, cudaStream_t st) {
  if (!setup_done_) throw std::invalid_argument("setup the network first");
  const Tensor& in = tensors_[input_t_];
  const long nimg = (long)batch_ * in_c_real_ * in.H * in.W;
  const float* src = images;
  if (from_host) {
    check(cudaMemcpyAsync(d_images_, images, nimg * 4, cudaMemcpyHostToDevice, st), "h2d images");
    src = d_images_;
  }
  check(cudaMemcpyAsync(d_labels_, labels, batch_ * 4, from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                        st),
        "labels");
  check(rfk::pack_input(src, batch_, in_c_real_, in.H, in.W, in.C, d_input_, st), "pack_input");
}

void Net::ensure_staging() {
  if (d_stage_images_[0]) return;
  const Tensor& in = tensors_[input_t_];
  const long nimg = (long)batch_ * in_c_real_ * in.H * in.W;
  for (int s = 0; s < 2; ++s) {
    check(cudaMalloc(&d_stage_images_[s], nimg * 4), "staging images");
    check(cudaMalloc(&d_stage_labels_[s], batch_ * 4), "staging labels");
    rep_.device_bytes += nimg * 4 + batch_ * 4;
    check(cudaEventCreateWithFlags(&stage_ready_[s], cudaEventDisableTiming), "event");
    check(cudaEventCreateWithFlags(&stage_free_[s], cudaEventDisableTiming), "event");
  }
}

void Net::stage_batch(const float* images_host, const int* labels_host, int slot, cudaStream_t copy_st) {
  if (!setup_done_) throw std::invalid_argument("setup the network first");
  if (slot < 0 || slot > 1) throw std::invalid_argument("staging slot must be 0 or 1");
  ensure_staging();
  const Tensor& in = tensors_[input_t_];
  const long nimg = (long)batch_ * in_c_real_ * in.H * in.W;
  check(cudaStreamWaitEvent(copy_st, stage_free_[slot], 0), "wait");  // previous batch of the slot consumed
  check(cudaMemcpyAsync(d_stage_images_[slot], images_host, nimg * 4, cudaMemcpyHostToDevice, copy_st), "h2d");
  check(cudaMemcpyAsync(d_stage_labels_[slot], labels_host, batch_ * 4, cudaMemcpyHostToDevice, copy_st), "h2d");
  check(cudaEventRecord(stage_ready_[slot], copy_st), "event");
}

void Net::use_batch(int slot, cudaStream_t st) {
  if (slot < 0 || slot > 1 || !d_stage_images_[slot]) throw std::invalid_argument("slot was never staged");
  const Tensor& in = tensors_[input_t_];
  check(cudaStreamWaitEvent(st, stage_ready_[slot], 0), "wait");
  check(rfk::copy_bytes(d_labels_, d_stage_labels_[slot], batch_ * 4L, st), "labels");  // a kernel, not a memcpy node
  check(rfk::pack_input(d_stage_images_[slot], batch_, in_c_real_, in.H, in.W, in.C, d_input_, st), "pack_input");
  check(cudaEventRecord(stage_free_[slot], st), "event");
}

void Net::set_comm(int nranks, int rank, const char id[128], long bucket_bytes) {
  if (!setup_done_) throw std::invalid_argument("setup the network before set_comm");
  auto c = std::make_unique<NcclComm>();
  std::string err;
  if (!c->init(nranks, rank, id, &err)) throw std::runtime_error(err);
  comm_ = std::move(c);
  if (!comm_stream_) check(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "comm stream");
  if (!comm_done_) check(cudaEventCreateWithFlags(&comm_done_, cudaEventDisableTiming), "event");
  bucket_floats_ = std::max(1L, bucket_bytes / 4);
  plan_buckets();
  {
    const char* e = std::getenv("RFK_COMM_SMS");
    comm_sm_reserve_ = e ? std::max(0, std::atoi(e)) : (nranks > 1 ? 16 : 0);
  }
  // every replica starts from rank 0's parameters and BN state (data-parallel
  // SGD: same model, averaged gradients), then refreshes its bf16 GEMM copies
  if (!comm_->broadcast(d_param_, (size_t)n_params_, 0, comm_stream_, &err) ||
      !comm_->broadcast(d_state_, (size_t)n_state_, 0, comm_stream_, &err))
    throw std::runtime_error(err);
  check(cudaMemsetAsync(d_mom_, 0, n_params_ * 4, comm_stream_), "memset");
  prep_weights(comm_stream_);
  check(cudaStreamSynchronize(comm_stream_), "parameter broadcast");
  for (auto& p : phase_exec_)
    if (p) {
      cudaGraphExecDestroy(p);
      p = nullptr;
    }
}

// Which gradient ranges become final after which backward instruction.
// Parameters sit in the flat buffer in op order, and the backward finishes
// them roughly in reverse; a bucket is the longest finished suffix not yet
// reduced, emitted once it holds bucket_floats_ or the backward is over.
void Net::plan_buckets() {
  buckets_.clear();
  const int np = (int)params_.size();
  std::vector<char> done(np, 0);
  std::vector<std::vector<int>> of_op(ops_.size());
  for (int i = 0; i < np; ++i) of_op[params_[i].op].push_back(i);
  int frontier = np, reduced = np;  // params [frontier, np) finished; [reduced, np) already in a bucket
  int last_bwd = -1;
  for (int k = 0; k < (int)sched_.size(); ++k)
    if (sched_[k].kind == InstrKind::Backward) last_bwd = k;
  auto off = [&](int i) { return i >= np ? n_params_ : params_[i].offset; };
  for (int k = 0; k < (int)sched_.size(); ++k) {
    if (sched_[k].kind != InstrKind::Backward) continue;
    for (int i : of_op[sched_[k].op]) done[i] = 1;
    while (frontier > 0 && done[frontier - 1]) --frontier;
    const bool last = k == last_bwd;
    if (frontier < reduced && (off(reduced) - off(frontier) >= bucket_floats_ || last)) {
      buckets_.push_back({k, off(frontier), off(reduced)});
      reduced = frontier;
    }
  }
  if (!comm_ && !buckets_for_sgd_) return;  // dry run (bucket_plan): no device events needed
  for (auto e : bucket_events_) cudaEventDestroy(e);
  bucket_events_.assign(buckets_.size(), nullptr);
  for (auto& e : bucket_events_) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
}

std::vector<std::array<long, 3>> Net::bucket_plan(long bucket_bytes) {
  if (!planned_) throw std::invalid_argument("plan the network first");
  const long saved = bucket_floats_;
  auto saved_b = buckets_;
  bucket_floats_ = std::max(1L, bucket_bytes / 4);
  if (!comm_) plan_buckets();
  else {
    auto keep = std::move(comm_);
    plan_buckets();
    comm_ = std::move(keep);
  }
  std::vector<std::array<long, 3>> out;
  for (const auto& b : buckets_) out.push_back({(long)b.after_instr, b.lo, b.hi});
  bucket_floats_ = saved;
  buckets_ = std::move(saved_b);
  return out;
}

// Bytes of the activation arena / gradient arena an instruction writes.
void Net::instr_writes(const Instr& ins, std::vector<std::pair<long, long>>& act,
                       std::vector<std::pair<long, long>>& grad) const {
  act.clear();
  grad.clear();
  const Op& op = ops_[ins.op];
  if (ins.kind == InstrKind::Forward) {
    auto put = [&](int t) {
      if (t != input_t_ && t != loss_t_ && slot_[t] >= 0) act.push_back({slot_[t], slot_[t] + tensors_[t].bytes()});
    };
    put(op.out);
    if (op.fused_bn >= 0) put(ops_[op.fused_bn].out);
  } else if (ins.kind == InstrKind::Backward) {
    for (int t : op.in)
      if (t != input_t_ && grad_slot_[t] >= 0) grad.push_back({grad_slot_[t], grad_slot_[t] + tensors_[t].bytes()});
  }
}

void Net::join_wgrad(cudaStream_t st) {
  if (!wgrad_pending_) return;
  check(cudaEventRecord(wgrad_join_, wgrad_stream_), "event");
  check(cudaStreamWaitEvent(st, wgrad_join_, 0), "wait");
  wgrad_reads_act_.clear();
  wgrad_reads_grad_.clear();
  wgrad_pending_ = false;
}

bool Net::forward_backward(cudaStream_t st, bool early_sgd) {
  if (!setup_done_) throw std::invalid_argument("setup the network first");
  im2col_holder_ = -1;  // a new batch: the stem's im2col is rebuilt by the first forward
  const bool dp = comm_ && comm_->ready() && comm_->nranks() > 0;
  // Early SGD (whole steps only): each gradient bucket -- the longest suffix
  // of the flat buffer whose parameters' backward (and pending weight-gradient
  // GEMMs) are complete -- is updated on the side stream right away (after
  // its all-reduce when data-parallel), overlapping the rest of the backward.
  // Safe because a parameter is never read again in a step after its own
  // backward (re-forwards precede it), and the update is elementwise, so the
  // results are bit-identical to one update pass at the end.
  static const bool early_on = !std::getenv("RFK_EARLY_SGD") || std::atoi(std::getenv("RFK_EARLY_SGD")) != 0;
  early_sgd = early_sgd && early_on;
  if (early_sgd && !dp && (!buckets_for_sgd_ || bucket_events_.size() != buckets_.size())) {
    static const long mb = std::getenv("RFK_SGD_BUCKET_MB") ? std::atol(std::getenv("RFK_SGD_BUCKET_MB")) : 16;
    buckets_for_sgd_ = true;
    bucket_floats_ = std::max(1L, (mb << 20) / 4);
    if (!comm_stream_) check(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "update stream");
    plan_buckets();
  }
  if (early_sgd) {
    long covered = 0;
    for (const auto& bk : buckets_) covered += bk.hi - bk.lo;
    if (covered != n_params_) early_sgd = false;  // not every parameter finishes in a bucket: one pass at the end
  }
  const bool bucketed = dp || early_sgd;
  size_t b = 0;
  std::vector<std::pair<long, long>> wa, wg;
  auto overlaps = [](const std::vector<std::pair<long, long>>& w, const std::vector<std::pair<long, long>>& r) {
    for (const auto& x : w)
      for (const auto& y : r)
        if (x.first < y.second && y.first < x.second) return true;
    return false;
  };
  static const bool trace = std::getenv("RFK_TRACE_JOIN") != nullptr;
  int joins_act = 0, joins_grad = 0;
  for (int k = 0; k < (int)sched_.size(); ++k) {
    if (wgrad_pending_) {
      instr_writes(sched_[k], wa, wg);
      const bool ja = overlaps(wa, wgrad_reads_act_), jg = overlaps(wg, wgrad_reads_grad_);
      if (ja || jg) {
        joins_act += ja;
        joins_grad += jg && !ja;
        join_wgrad(st);
      }
    }
    run_instr(sched_[k], st);
    while (bucketed && b < buckets_.size() && buckets_[b].after_instr == k) {
      // the bucket's weight gradients must be complete: the comm stream (not
      // this one) waits for the pending side-stream weight-gradient GEMMs, so
      // the backward keeps going; the wgrad read sets stay pending for the
      // main stream's own lazy join
      if (wgrad_pending_) {
        check(cudaEventRecord(wgrad_join_, wgrad_stream_), "event");
        check(cudaStreamWaitEvent(comm_stream_, wgrad_join_, 0), "wait");
      }
      // fork: the side stream waits for the gradients, then reduces them
      // while this stream carries on with the backward
      check(cudaEventRecord(bucket_events_[b], st), "event");
      check(cudaStreamWaitEvent(comm_stream_, bucket_events_[b], 0), "wait");
      const long lo = buckets_[b].lo, n = buckets_[b].hi - buckets_[b].lo;
      if (dp) {
        comm_inflight_ = true;
        std::string err;
        if (!comm_->allreduce_avg(d_grad_ + lo, (size_t)n, comm_stream_, &err)) throw std::runtime_error(err);
      }
      if (early_sgd)
        check(rfk::sgd_update(d_param_ + lo, d_grad_ + lo, d_mom_ + lo, n, d_hyper_, d_bf16_ + lo, comm_stream_),
              "sgd");
      ++b;
    }
  }
  join_wgrad(st);
  comm_inflight_ = false;
  if (trace)
    std::fprintf(stderr, "wgrad joins: %d on activation ranges, %d on gradient ranges; %zu buckets, early SGD %d\n",
                 joins_act, joins_grad, b, (int)early_sgd);
  if (bucketed) {  // join
    if (!comm_done_) check(cudaEventCreateWithFlags(&comm_done_, cudaEventDisableTiming), "event");
    check(cudaEventRecord(comm_done_, comm_stream_), "event");
    check(cudaStreamWaitEvent(st, comm_done_, 0), "wait");
  }
  return early_sgd;
}

// SGD hyperparameters live in device memory (d_hyper_ = {lr, momentum, wd}),
// written in stream order before each step, so one captured step graph
// serves any learning-rate schedule.  The source is pageable: cudaMemcpyAsync
// stages it before returning, so the stack buffer may go away.
// Unchanged values are not re-sent (a constant schedule then launches the
// step graph back to back, without a copy in between).
void Net::set_hyper(float lr, float momentum, float wd, cudaStream_t st) {
  const float h[3] = {lr, momentum, wd};
  if (hyper_valid_ && std::memcmp(h, hyper_last_, sizeof h) == 0) return;
  check(cudaMemcpyAsync(d_hyper_, h, sizeof h, cudaMemcpyHostToDevice, st), "hyper h2d");
  std::memcpy(hyper_last_, h, sizeof h);
  hyper_valid_ = true;
}

void Net::update(cudaStream_t st) {
  // one pass: momentum SGD on the fp32 masters + refresh of their bf16 copy
  check(rfk::sgd_update(d_param_, d_grad_, d_mom_, n_params_, d_hyper_, d_bf16_, st), "sgd");
}

cudaGraphExec_t Net::capture(const std::function<void(cudaStream_t)>& body, long* kernel_nodes) {
  cudaStream_t cap;
  create_stream(&cap, true);  // capture (main path) stream
  check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
  try {
    body(cap);
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(cap, &g);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    throw;
  }
  cudaGraph_t g;
  check(cudaStreamEndCapture(cap, &g), "end capture");
  size_t nn = 0;
  check(cudaGraphGetNodes(g, nullptr, &nn), "graph nodes");
  std::vector<cudaGraphNode_t> nodes(nn);
  check(cudaGraphGetNodes(g, nodes.data(), &nn), "graph nodes");
  long kernels = 0;
  for (auto n : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(n, &t);
    if (t == cudaGraphNodeTypeKernel) ++kernels;
  }
  if (kernel_nodes) *kernel_nodes = kernels;
  cudaGraphExec_t exec = nullptr;
  check(cudaGraphInstantiate(&exec, g, prio_enabled() ? cudaGraphInstantiateFlagUseNodePriority : 0), "instantiate");
  cudaGraphDestroy(g);
  cudaStreamDestroy(cap);
  return exec;
}

void Net::run_phase(int phase, float lr, float momentum, float wd, cudaStream_t st, bool use_graph) {
  auto body = [&](cudaStream_t s) {
    bool updated = false;
    if (phase == 0 || phase == 2) updated = forward_backward(s, phase == 2);
    if ((phase == 1 || phase == 2) && !updated) update(s);
  };
  if (phase == 1 || phase == 2) set_hyper(lr, momentum, wd, st);
  if (!use_graph) {
    body(st);
    return;
  }
  if (!phase_exec_[phase]) {
    long k = 0;
    phase_exec_[phase] = capture(body, &k);
    if (phase == 2) rep_.launches_per_step = k;
  }
  check(cudaGraphLaunch(phase_exec_[phase], st), "graph launch");
}

void Net::step(float lr, float momentum, float wd, cudaStream_t st, bool use_graph) {
  run_phase(2, lr, momentum, wd, st, use_graph);
}

std::vector<std::array<double, 10>> Net::gemm_profile_detail(int iters, cudaStream_t st) {
  double a, b;
  long c;
  if (gemm_trace_.empty()) gemm_profile(1, st, &a, &b, &c);
  // the whole GEMM list as one CUDA graph with an event node after every
  // launch: device times in step order, no host launch overhead
  const size_t n = gemm_trace_.size();
  std::vector<cudaEvent_t> ev(n + 1);
  for (auto& e : ev) check(cudaEventCreate(&e), "event");
  cudaGraphExec_t g = capture(
      [&](cudaStream_t s) {
        check(cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal), "event");
        for (size_t i = 0; i < n; ++i) {
          check(rfk::gemm_launch(gemm_trace_[i].desc, s), "gemm");
          check(cudaEventRecordWithFlags(ev[i + 1], s, cudaEventRecordExternal), "event");
        }
      },
      nullptr);
  std::vector<double> ms(n, 0.0);
  for (int it = 0; it < iters + 1; ++it) {
    check(cudaGraphLaunch(g, st), "graph");
    check(cudaStreamSynchronize(st), "sync");
    if (it == 0) continue;  // warm-up
    for (size_t i = 0; i < n; ++i) {
      float t = 0;
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
      ms[i] += t / iters;
    }
  }
  cudaGraphExecDestroy(g);
  for (auto e : ev) cudaEventDestroy(e);
  std::vector<std::array<double, 10>> out;
  for (size_t i = 0; i < n; ++i) {
    const auto& d = gemm_trace_[i].desc;
    out.push_back({(double)d.M, (double)d.N, (double)d.K, (double)(int)d.a_kind, (double)(int)d.b_kind,
                   (double)d.splits, ms[i], gemm_trace_[i].flops, gemm_trace_[i].bytes,
                   (double)rfk::gemm_block_n(d)});
  }
  return out;
}

void Net::gemm_profile(int iters, cudaStream_t st, double* ms_per_step, double* flops_per_step, long* launches) {
  if (gemm_trace_.empty()) {
    tracing_ = true;
    try {
      cudaGraphExec_t e = capture([&](cudaStream_t s) { forward_backward(s); }, nullptr);
      cudaGraphExecDestroy(e);  // only the trace was wanted
    } catch (...) {
      tracing_ = false;
      throw;
    }
    tracing_ = false;
  }
  double flops = 0;
  for (const auto& r : gemm_trace_) flops += r.flops;
  cudaGraphExec_t g = capture(
      [&](cudaStream_t s) {
        for (const auto& r : gemm_trace_) check(rfk::gemm_launch(r.desc, s), "gemm");
      },
      nullptr);
  cudaEvent_t e0, e1;
  check(cudaEventCreate(&e0), "event");
  check(cudaEventCreate(&e1), "event");
  for (int i = 0; i < 2; ++i) check(cudaGraphLaunch(g, st), "warmup");
  check(cudaEventRecord(e0, st), "event");
  for (int i = 0; i < iters; ++i) check(cudaGraphLaunch(g, st), "gemm replay");
  check(cudaEventRecord(e1, st), "event");
  check(cudaEventSynchronize(e1), "event sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(g);
  *ms_per_step = ms / iters;
  *flops_per_step = flops;
  *launches = (long)gemm_trace_.size();
}

double Net::gemm_try(int idx, int block_n, int splits, int iters, cudaStream_t st) {
  if (gemm_trace_.empty()) {
    double a, b;
    long c;
    gemm_profile(1, st, &a, &b, &c);
  }
  if (idx < 0 || idx >= (int)gemm_trace_.size()) throw std::invalid_argument("gemm index out of range");
  rfk::GemmDesc d = gemm_trace_[idx].desc;
  d.block_n = block_n;
  d.splits = splits < 1 ? 1 : splits;
  d.stats = nullptr;
  d.stats_bwd = false;
  d.bias = nullptr;
  d.remap = false;
  d.accumulate_out = false;
  d.out_f32 = true;
  d.ldc = d.N;
  d.split_stride = (long)d.M * d.N;
  void* scratch = nullptr;
  check(cudaMalloc(&scratch, (size_t)d.splits * d.M * d.N * 4), "scratch");
  d.out = scratch;
  // device time: `iters` launches captured in one CUDA graph (no host
  // tensor-map encoding or launch overhead between them)
  cudaGraphExec_t g = capture(
      [&](cudaStream_t s) {
        for (int i = 0; i < iters; ++i) check(rfk::gemm_launch(d, s), "gemm");
      },
      nullptr);
  cudaEvent_t e0, e1;
  check(cudaEventCreate(&e0), "event");
  check(cudaEventCreate(&e1), "event");
  check(cudaGraphLaunch(g, st), "warmup");
  check(cudaEventRecord(e0, st), "event");
  check(cudaGraphLaunch(g, st), "graph");
  check(cudaEventRecord(e1, st), "event");
  check(cudaEventSynchronize(e1), "sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaGraphExecDestroy(g);
  cudaFree(scratch);
  return ms / iters;
}

std::vector<double> Net::instr_profile(int iters, cudaStream_t st) {
  if (!setup_done_) throw std::invalid_argument("setup the network first");
  // the step as one CUDA graph with an event node after every instruction:
  // in-graph device times, no host launch overhead
  const size_t n = sched_.size();
  std::vector<cudaEvent_t> ev(n + 2);
  for (auto& e : ev) check(cudaEventCreate(&e), "event");
  cudaGraphExec_t g = capture(
      [&](cudaStream_t s) {
        check(cudaEventRecordWithFlags(ev[0], s, cudaEventRecordExternal), "event");
        im2col_holder_ = -1;  // as in forward_backward
        for (size_t k = 0; k < n; ++k) {
          run_instr(sched_[k], s);
          join_wgrad(s);  // per-instruction attribution: no cross-instruction overlap
          check(cudaEventRecordWithFlags(ev[k + 1], s, cudaEventRecordExternal), "event");
        }
        update(s);  // hyperparameters zeroed below: parameters unchanged
        check(cudaEventRecordWithFlags(ev[n + 1], s, cudaEventRecordExternal), "event");
      },
      nullptr);
  std::vector<double> ms(n + 1, 0.0);
  set_hyper(0.f, 0.f, 0.f, st);  // lr 0
  for (int it = 0; it < iters + 1; ++it) {
    check(cudaGraphLaunch(g, st), "graph");
    check(cudaStreamSynchronize(st), "sync");
    if (it == 0) continue;  // warm-up
    for (size_t k = 0; k <= n; ++k) {
      float t = 0;
      cudaEventElapsedTime(&t, ev[k], ev[k + 1]);
      ms[k] += t / iters;
    }
  }
  cudaGraphExecDestroy(g);
  for (auto e : ev) cudaEventDestroy(e);
  return ms;
}

void Net::copy_loss(float* dst, cudaStream_t st) {
  check(cudaMemcpyAsync(dst, d_loss_, 4, cudaMemcpyDeviceToHost, st), "loss d2h");
}

float Net::read_loss(cudaStream_t st) {
  float v = 0.f;
  check(cudaMemcpyAsync(&v, d_loss_, 4, cudaMemcpyDeviceToHost, st), "loss d2h");
  check(cudaStreamSynchronize(st), "sync");
  return v;
}

}  // namespace rfx
