// Re-forward training executor: network IR, plan, schedule and runtime.
//
// A network is a DAG of ops over activation tensors (NHWC bf16; logits fp32).
// Its tensor graph — vertex = tensor, cost = its arena bytes, edge = op
// input -> output — is exactly the computation graph of the paper (§4 "the
// vertices represent the DNN tensors and the edges represent DNN
// operations"), handed to the host planner (reforward::solve_acg).  The plan's
// stored set V^R gets fixed slots in the activation arena; every segment (a
// weakly-connected component of non-stored tensors) is packed into one shared
// re-forward region sized to the largest segment, so the arena is
// stored_cost + max_segment = Eq. 1, and the schedule's live-byte high-water
// mark is tracked to prove it.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "executor/comm.h"
#include "kernels/kernels.h"
#include "kernels/ops.h"

namespace rfx {

enum class DType : int { BF16 = 0, F32 = 1 };
enum class OpKind : int { Input = 0, Conv, BN, BNAddReLU, ReLU, MaxPool, AvgPool, FC, Concat, Loss, AvgPool2d, Linear };
const char* op_kind_name(OpKind k);

constexpr long kAlign = 1024;  // arena slot alignment (bytes); costs are rounded to it
constexpr long kStatRows = 160;
constexpr long kArenaGuard = 1 << 20;  // canary bytes behind the activation arena  // fused-BN partial rows: >= the persistent GEMM grid (SM count)
inline long align_up(long x, long a = kAlign) { return (x + a - 1) / a * a; }

struct Tensor {
  std::string name;
  int N = 0, H = 1, W = 1, C = 0;
  DType dtype = DType::BF16;
  int producer = -1;
  std::vector<int> consumers;
  long elems() const { return (long)N * H * W * C; }
  long bytes() const { return elems() * (dtype == DType::BF16 ? 2 : 4); }
  long cost() const { return align_up(bytes()); }  // planner vertex cost
  long rows() const { return (long)N * H * W; }
};

struct BNState {  // per-BN-layer device state (persistent, fp32 [C] each)
  int C = 0;
  long mean = 0, invstd = 0, scale = 0, shift = 0, run_mean = 0, run_var = 0, coef = 0;  // offsets (floats)
};

struct Param {
  std::string name;
  int kind = 0;  // 0 conv weight, 1 bn gamma, 2 bn beta, 3 fc weight, 4 fc / linear bias, 5 linear weight
  int op = -1;
  long offset = 0, count = 0;          // slice of the flat fp32 master / grad / momentum buffers
  long bf16_off = -1, bf16_count = 0;  // bf16 GEMM-layout copy (conv / fc weights)
  long wt_off = -1, wt_count = 0;      // bf16 flipped transpose for conv dgrad
  std::vector<int> shape;              // canonical (PyTorch) shape
};

struct Op {
  OpKind kind = OpKind::Input;
  std::string name;
  std::vector<int> in;
  int out = -1;
  // conv
  int R = 1, S = 1, stride = 1, pad = 0;  // pad = height padding (and width unless pad_w is set)
  int pad_w = 0;
  int cin = 0, cin_real = 0, cout = 0, cpad = 0, coutpad = 0;
  bool explicit_im2col = false;
  int kpad = 0;              // explicit im2col K (padded)
  int im2col_imgs = 0;       // images per explicit-im2col chunk (the chunk stays in L2)
  bool fuse_stats = false;   // conv epilogue emits BN partial sums for its consumer
  long stats_off = -1;       // its slot in the statistics workspace (floats)
  int wg_splits = 1, wg_bn = 128;  // wgrad split-K and tile N
  int fp_splits = 1, fp_bn = 0;    // fprop split-K (bf16 finish kernel) and tile N
  int dg_splits = 1, dg_bn = 0;    // dgrad split-K and tile N
  bool dg_subpixel = false;        // strided dgrad as s*s stride-1 sub-pixel GEMMs (no zero insertion)
  int fused_bn = -1;               // conv: BN op whose re-forward runs in this conv's epilogue
  bool reforward_in_producer = false;  // BN: re-forwarded by its producing conv's epilogue
  int bn_gather = -1;              // BN over a concatenation: index of its statistics-gather table
  // BN+ReLU backward statistics from rows (sum g, sum g*(y-mean)) written by
  // the consumer conv's dgrad epilogue when the BN input is resident at that
  // point (bstat_fused), else by a replay over the stored dout at the BN's
  // backward -- same tiles, same CTAs, so the rows are plan-independent
  bool bstat = false;              // BN: backward statistics from rows
  bool bstat_resident = false;     // BN: input resident at the consumer conv's backward (schedule)
  bool bstat_fused = false;        // BN: rows produced by the consumer conv's dgrad epilogue
  long bstat_off = -1;             // BN: its rows slot in the statistics workspace (floats)
  int bstat_bn = 0;                // BN: tile width of the rows (the dgrad's, fixed)
  int bstat_src = -1;              // conv: BN whose rows its dgrad epilogue produces
  // pool
  int k = 1;
  long pool_idx_off = -1;  // max pool: its argmax slot (bytes) in the pool-index workspace region
  // classifier / linear
  int classes = 0;  // output features
  int lin_h = 1, lin_w = 1, lin_c = 0;  // linear: input spatial shape (flattened NHWC)
  // parameters / state
  int w_param = -1, b_param = -1;  // conv/fc weight + fc bias; bn gamma (w) + beta (b)
  int bn = -1;                     // BNState index
  float eps = 1e-5f, momentum = 0.1f;
};

struct Plan {
  std::string policy;
  std::vector<char> stored;   // per tensor
  std::vector<int> seg_of;    // per tensor, -1 unless in a segment
  std::vector<long> seg_cost;
  long stored_cost = 0, max_seg = 0, total = 0, store_all_total = 0, candidate_max_term = 0;
};

enum class InstrKind : int { Forward = 0, Backward = 1, Release = 2 };
struct Instr {
  InstrKind kind;
  int op = -1;
  int seg = -1;
  bool reforward = false;
  int phase = 0;  // two-phase forward of an add/concat whose inputs sit in two segments
};

struct MemoryReport {
  long planned_total = 0;       // Eq. 1 of the plan (stored + max segment)
  long stored_cost = 0, max_segment = 0, store_all_total = 0;
  long tracked_peak = 0;        // high-water mark of live activation bytes over the schedule
  long arena_bytes = 0;         // activation arena capacity
  long grad_arena_bytes = 0, workspace_bytes = 0, param_bytes = 0, state_bytes = 0;
  long reforward_ops = 0, segment_loads = 0, forward_ops = 0, backward_ops = 0;
  long launches_per_step = 0;
  long device_bytes = 0;  // every cudaMalloc of this net (arena + guard, gradients, workspace, parameters, ...)
};

struct SubpixelDim {
  int r0 = 0, J = 0, c = 0, pad_lo = 0, rows = 0;
};
SubpixelDim subpixel_dim(int a, int stride, int R, int pad, int H);

class Net;
std::unique_ptr<Net> make_net(int batch);

class Net {
 public:
  explicit Net(int batch) : batch_(batch) {}
  ~Net();

  // ---------------------------------------------------------- building
  int input(int H, int W, int C);  // NCHW fp32 images -> NHWC bf16 (C padded to 8)
  int conv(int x, int cout, int R, int S, int stride, int pad, const std::string& name);
  // rectangular padding (Inception's 1x7 / 7x1 / 1x3 / 3x1 convolutions)
  int conv2(int x, int cout, int R, int S, int stride, int pad_h, int pad_w, const std::string& name);
  int bn(int y, bool relu, const std::string& name);
  int bn_add_relu(int y, int skip, const std::string& name);
  int relu(int x, const std::string& name);
  int maxpool(int x, int k, int stride, int pad, const std::string& name);
  int avgpool(int x, const std::string& name);                                     // global
  int avgpool2d(int x, int k, int stride, int pad, const std::string& name);       // windowed
  int fc(int x, int classes, const std::string& name);                             // fp32 logits
  int linear(int x, int out_features, const std::string& name);                    // bf16 hidden layer
  int concat(int a, int b, const std::string& name);
  int loss(int logits, const std::string& name);

  // ---------------------------------------------------------- planning
  // policy: "reforward" (Algorithm 5 / solve_acg), "store_all", "lcg"
  // (Algorithm 1, linear graphs), "sqrt" (even sqrt(N) heuristic, linear).
  void plan(const std::string& policy);
  void plan_with_stored(const std::vector<char>& stored, const std::string& label);
  void graph_export(std::vector<std::string>& names, std::vector<long>& costs,
                    std::vector<std::pair<int, int>>& edges) const;

  // ---------------------------------------------------------- runtime
  void setup(uint64_t seed);  // allocate device memory, init parameters
  void load_batch(const float* images, const int* labels, bool from_host, cudaStream_t st);
  // Double-buffered input pipeline: stage_batch copies a host batch (pinned
  // for overlap) into staging slot 0/1 on `copy_st` once the slot's previous
  // batch has been consumed; use_batch makes `st` wait for the slot, packs it
  // into the network input and releases the slot.  Staging batch k+1 while
  // step k runs hides the host->device copy behind the step.
  void stage_batch(const float* images_host, const int* labels_host, int slot, cudaStream_t copy_st);
  void use_batch(int slot, cudaStream_t st);
  // loss + gradients; with early_sgd, also the momentum SGD of every gradient
  // bucket as soon as the backward has finalised it (returns whether it did)
  bool forward_backward(cudaStream_t st, bool early_sgd = false);
  void update(float lr, float momentum, float wd, cudaStream_t st) {  // SGD + weight prep
    set_hyper(lr, momentum, wd, st);
    update(st);
  }
  void set_hyper(float lr, float momentum, float wd, cudaStream_t st);
  void update(cudaStream_t st);  // SGD with the device-resident hyperparameters
  void step(float lr, float momentum, float wd, cudaStream_t st, bool use_graph);
  // phase: 0 forward+backward, 1 update, 2 both (each cached as its own CUDA graph)
  void run_phase(int phase, float lr, float momentum, float wd, cudaStream_t st, bool use_graph);
  void copy_loss(float* dst, cudaStream_t st);  // async D2H (dst pinned: no host sync)
  float read_loss(cudaStream_t st);

  // Live roofline probe of the dense-contraction kernels: replay exactly the
  // GEMM launches of one step (same shapes, same buffers) as a CUDA graph and
  // time it with events.  flops = algorithmic 2*M*N*K of the real (unpadded)
  // problem summed over those launches.
  void gemm_profile(int iters, cudaStream_t st, double* ms_per_step, double* flops_per_step, long* launches);
  // per-launch timing of the step's GEMMs (events between eager launches):
  // rows of {M, N, K, a_kind, b_kind, splits, ms, flops}
  std::vector<std::array<double, 10>> gemm_profile_detail(int iters, cudaStream_t st);
  // in-stream time of every schedule instruction (events between eager
  // launches, averaged over iters) followed by the SGD update: size = |schedule| + 1
  std::vector<double> instr_profile(int iters, cudaStream_t st);
  // tuning probe: re-time traced GEMM `idx` with a forced tile width and
  // split count (fp32 partials into a scratch buffer; the step's buffers are
  // not written)
  double gemm_try(int idx, int block_n, int splits, int iters, cudaStream_t st);

  // parameter access in canonical layout (host fp32)
  int num_params() const { return (int)params_.size(); }
  const Param& param(int i) const { return params_[i]; }
  void read_param(int i, int which, float* host) const;  // which: 0 value, 1 grad, 2 momentum
  void write_param(int i, const float* host);
  // host-only layout conversion: canonical <-> the slice [param_offset(i),
  // + param_count(i)) of the flat fp32 parameter / gradient buffers
  void pack_param(int i, const float* canonical, float* flat_slice) const;
  float* ws_stats_base() const;  // BN statistics rows region of the workspace
  uint8_t* pool_idx(const Op& op) const;  // a max pool's argmax slot (nullptr: none)
  void unpack_param(int i, const float* flat_slice, float* canonical) const;
  long param_offset(int i) const { return params_.at(i).offset; }
  long param_count(int i) const { return params_.at(i).count; }
  void read_tensor(int t, float* host) const;
  void read_grad_tensor(int t, float* host) const;  // valid for every tensor with keep_grads
  void set_keep_grads(bool on) { keep_grads_ = on; }
  void read_bn_running(int op, float* mean, float* var) const;

  float* grad_buffer() const { return d_grad_; }
  // true when the canary band behind the Eq.-1-sized activation arena is untouched
  bool arena_guard_intact() const;
  long grad_count() const { return n_params_; }

  // Data parallel: average the flat gradient buffer across ranks with NCCL,
  // bucket by bucket as the backward finalises parameter gradients (on a
  // side stream, overlapped with the remaining backward; captured into the
  // step's CUDA graph like everything else).
  void set_comm(int nranks, int rank, const char id[128], long bucket_bytes);
  int comm_buckets() const { return (int)buckets_.size(); }
  // dry run of the bucket plan: (after instruction, lo, hi) per bucket
  std::vector<std::array<long, 3>> bucket_plan(long bucket_bytes);

  const MemoryReport& report() const { return rep_; }
  const Plan& current_plan() const { return plan_; }
  const std::vector<Tensor>& tensors() const { return tensors_; }
  const std::vector<Op>& ops() const { return ops_; }
  const std::vector<Instr>& schedule() const { return sched_; }
  int batch() const { return batch_; }
  long flops_per_step() const;

 private:
  int add_tensor(const std::string& name, int N, int H, int W, int C, DType dt);
  int add_op(Op op);
  int add_param(const std::string& name, int kind, int op, long count, std::vector<int> shape);
  void build_schedule();
  void layout();
  void run_instr(const Instr& ins, cudaStream_t st);
  void op_forward(const Op& op, bool reforward, int phase, cudaStream_t st);
  void op_backward(const Op& op, cudaStream_t st);
  void prep_weights(cudaStream_t st);
  void prep_weights_table(cudaStream_t st);  // per-layer table variant (unused by the step)
  void* tptr(int t) const;
  __nv_bfloat16* tb(int t) const { return static_cast<__nv_bfloat16*>(tptr(t)); }
  __nv_bfloat16* gptr(int t) const;
  void gemm(const rfk::GemmDesc& d, cudaStream_t st);
  bool wgrad_overlap() const;
  bool subpixel_ok(const Op& op, const Tensor& x) const;  // strided dgrad as sub-pixel GEMMs
  bool fusable_conv(const Op& op) const;  // some plan may fuse its consumer BN into its re-forward
  void ensure_wgrad_stream();
  void ensure_sub_streams();
  void check(cudaError_t e, const char* what) const;
  void free_device();

  int batch_;
  std::vector<Tensor> tensors_;
  std::vector<Op> ops_;
  std::vector<Param> params_;
  std::vector<BNState> bns_;
  int input_t_ = -1, loss_t_ = -1, logits_t_ = -1;
  int in_c_real_ = 0;
  long n_params_ = 0, n_bf16_ = 0, n_state_ = 0;

  Plan plan_;
  bool planned_ = false;
  bool keep_grads_ = false;
  std::vector<Instr> sched_;
  std::vector<long> slot_;        // arena offset per tensor (stored or segment slot)
  std::vector<long> grad_slot_;   // grad arena offset per tensor, -1 if none
  std::vector<char> grad_acc_;    // per (op, input) accumulate flags, flattened
  std::vector<int> grad_acc_base_;
  long arena_bytes_ = 0, grad_bytes_ = 0;
  long ws_pool_ = 0;  // per-max-pool argmax bytes, after ws_dsplit_ (written by every forward of the pool)
  long ws_im2col_ = 0, ws_partials_ = 0, ws_zero_ = 0, ws_split_ = 0, ws_stats_ = 0, ws_misc_ = 0,
       ws_counters_ = 0, ws_dsplit_ = 0;
  MemoryReport rep_;
  long launches_ = 0;
  bool counting_ = false;

  // device memory
  bool setup_done_ = false;
  uint8_t* d_arena_ = nullptr;
  uint8_t* d_grad_arena_ = nullptr;
  uint8_t* d_ws_ = nullptr;
  float* d_param_ = nullptr;
  float* d_grad_ = nullptr;
  float* d_mom_ = nullptr;
  __nv_bfloat16* d_bf16_ = nullptr;
  float* d_state_ = nullptr;
  __nv_bfloat16* d_input_ = nullptr;
  float* d_images_ = nullptr;
  float* d_stage_images_[2] = {nullptr, nullptr};
  int* d_stage_labels_[2] = {nullptr, nullptr};
  cudaEvent_t stage_ready_[2] = {nullptr, nullptr}, stage_free_[2] = {nullptr, nullptr};
  void ensure_staging();
  int* d_labels_ = nullptr;
  float* d_loss_ = nullptr;
  float* d_rowloss_ = nullptr;
  float* d_lse_ = nullptr;
  float* d_hyper_ = nullptr;
  float hyper_last_[3] = {0.f, 0.f, 0.f};  // last values uploaded to d_hyper_
  bool hyper_valid_ = false;
  cudaGraphExec_t graph_exec_ = nullptr;
  float graph_lr_ = 0, graph_mom_ = 0, graph_wd_ = 0;
  cudaGraphExec_t phase_exec_[3] = {nullptr, nullptr, nullptr};
  std::unique_ptr<NcclComm> comm_;
  cudaStream_t comm_stream_ = nullptr;
  // conv backward: the weight-gradient GEMM runs on a side stream next to the
  // data-gradient GEMM (fork / join inside the step graph)
  cudaStream_t wgrad_stream_ = nullptr;
  cudaEvent_t wgrad_fork_ = nullptr, wgrad_join_ = nullptr;
  // sub-pixel dgrad: class GEMMs 1..3 run on their own streams next to class 0
  cudaStream_t sub_stream_[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t sub_fork_ = nullptr, sub_join_[3] = {nullptr, nullptr, nullptr};
  bool wgrad_pending_ = false;
  std::vector<std::pair<long, long>> wgrad_reads_act_, wgrad_reads_grad_;  // byte ranges pending wgrads read
  void instr_writes(const Instr& ins, std::vector<std::pair<long, long>>& act,
                    std::vector<std::pair<long, long>>& grad) const;
  void join_wgrad(cudaStream_t st);
  struct Bucket {
    int after_instr;  // launch once this schedule instruction has been enqueued
    long lo, hi;      // float range of the gradient buffer
  };
  std::vector<Bucket> buckets_;
  std::vector<cudaEvent_t> bucket_events_;
  cudaEvent_t comm_done_ = nullptr;
  long bucket_floats_ = 0;
  bool buckets_for_sgd_ = false;  // buckets_ planned without a communicator (early SGD)
  void plan_buckets();
  void* d_prep_table_ = nullptr;
  // BN over concatenations (DenseNet): per BN, the concat's leaf tensors in
  // channel order; per leaf, its partial-sum slot (floats into the stats
  // workspace) and row count; one device table of 32-channel blocks
  std::vector<std::vector<int>> gather_leaves_;
  std::vector<long> leaf_stats_off_;   // per tensor; -1 = not a colstats leaf
  std::vector<int> gather_first_block_;
  void* d_gather_ = nullptr;
  void build_gather_tables();
  int prep_layers_ = 0;
  long prep_total_ = 0;

  struct GemmRecord {
    rfk::GemmDesc desc;
    double flops;
    double bytes;  // algorithmic HBM bytes: operands read once + output written (read too when accumulating)
  };
  bool tracing_ = false;
  // a gradient bucket's all-reduce may be running on comm_stream_: persistent
  // GEMMs leave comm_sm_reserve_ SMs to the NCCL kernels (RFK_COMM_SMS)
  bool comm_inflight_ = false;
  int comm_sm_reserve_ = 0;
  bool tuned_ = false;
  int im2col_holder_ = -1;  // explicit-im2col conv whose whole-batch matrix ws_im2col holds (this step)
  void autotune(cudaStream_t st);  // per GEMM shape: fastest tile width (process-wide cache)
  double trace_flops_ = 0;  // algorithmic flops to attach to the next traced GEMM
  std::vector<GemmRecord> gemm_trace_;
  cudaGraphExec_t capture(const std::function<void(cudaStream_t)>& body, long* kernel_nodes);

  friend class Scheduler;
};

}  // namespace rfx
