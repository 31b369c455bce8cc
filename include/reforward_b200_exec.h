/* Executor / kernel half of the C-ABI (see reforward_b200.h for conventions).
 * No reference counterpart: these are the train-step entry points the
 * reference's plan drives. */
#ifndef REFORWARD_B200_EXEC_H_
#define REFORWARD_B200_EXEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ raw GEMM engine
 * D[M,N] = sum_k A[m,k] B[n,k] on tcgen05 (bf16 in, fp32 accumulate).
 * kind: 0 K-major 2-D, 1 MN-major 2-D, 2 im2col (K-major), 3 im2col (MN-major). */
typedef struct rfx_conv_geom {
  int32_t N, H, W, C, P, Q, R, S, pad_h, pad_w, stride_h, stride_w;
} rfx_conv_geom;

typedef struct rfx_gemm_args {
  int32_t M, N, K;
  int32_t a_kind;
  const void* a;
  int64_t a_ld;
  rfx_conv_geom a_geom;
  int32_t b_kind;
  const void* b;
  int64_t b_ld;
  rfx_conv_geom b_geom;
  void* out;
  int64_t ldc;
  int32_t out_f32;
  int32_t accumulate_out;
  const float* bias;
  float* stats;
  int32_t splits;
  int64_t split_stride;
  int32_t remap, rP, rQ, rH, rW, rsh, rsw;
  int32_t block_n;
  int64_t b_extent;                  /* valid MN extent of an MN-major B (0 = N) */
  int32_t b_taps, b_cpad, b_rows;    /* kind 4 (conv weights as dgrad B): R*S, Cpad, Cout */
  int32_t band;                      /* stride-1 im2col A: nonzero = the shifted-band kernel wherever the shape and
                                      * epilogue allow it (the executor uses it only where it measured faster);
                                      * with one 64-channel block of A its bits equal the im2col kernel's */
  int32_t b_tap_map;                 /* kind 4: nonzero = weight tap of A tap (r, s) is base - r*dr - s*ds */
  int32_t b_tap_base, b_tap_dr, b_tap_ds;  /* (sub-pixel dgrad classes); zero = flipped full filter */
  /* BN+ReLU backward statistics in the epilogue (with `stats`): out (dout of
   * the BN+ReLU output) is stored as is; stats rows [CTA][2][N] hold sum g and
   * sum g*(y - mean), g = dout * [y*scale + shift > 0].  replay: no GEMM, the epilogue re-reads `out` (a fixed
   * block_n is required) and writes bit-identical rows. */
  int32_t stats_bwd, replay;
  const void* bs_y;                  /* bf16 [M][bs_ldy], the BN input */
  int64_t bs_ldy;
  const float* bs_mean;
  const float* bs_scale;
  const float* bs_shift;
  int32_t pair;                      /* CTA pairs (cta_group::2, M = 256): 0 auto, 1 where allowed, -1 never */
} rfx_gemm_args;
/* kind 4 = conv weights [Cout][R][S][Cpad] read as the dgrad B operand (flipped taps) */

int rfx_gemm(const rfx_gemm_args* args, void* stream);
/* sizeof(rfx_gemm_args) as compiled: lets FFI callers check their layout */
size_t rfx_gemm_args_size(void);
/* explicit im2col of a few-channel NHWC bf16 conv input (the stem path):
 * x [N][H][W][Cs] (C real channels) -> out [N*P*Q][kpad], K order (r, s, c),
 * zero K padding; kpad % 8 == 0 */
/* max-pool backward (NHWC bf16, C % 8 == 0): dx (+)= sum over the windows
 * whose first argmax is the pixel of their dy, in fixed window order.
 * workspace: N*P*Q*C bytes, used only by the two-pass fallback */
int rfx_maxpool_bwd(const void* x, const void* dy, int N, int H, int W, int C, int k, int stride, int pad, void* dx,
                    int accumulate, void* workspace, void* stream);
int rfx_im2col(const void* x, int N, int H, int W, int C, int Cs, int P, int Q, int R, int S, int stride, int pad,
               int kpad, void* out, void* stream);

/* ------------------------------------------------------------ re-forward training executor
 * A network is a DAG of ops over NHWC tensors; each builder call returns the
 * id of the op's output tensor.  rfx_net_plan runs the host planner on the
 * tensor graph (vertex = tensor, cost = arena bytes) and derives the
 * re-forward schedule and arena layout; rfx_net_setup allocates device memory.
 * Streams are cudaStream_t passed as void* (NULL = legacy default stream). */
typedef struct rfx_net rfx_net;

int rfx_net_create(int32_t batch, rfx_net** out);
/* arch: resnet18..152, densenet121/161/169/201, densenet_tiny, vgg11..19, alexnet, inception_v3, chain8 */
int rfx_net_create_named(const char* arch, int32_t batch, int32_t H, int32_t W, int32_t classes,
                         rfx_net** out);
void rfx_net_free(rfx_net* net);

int rfx_net_input(rfx_net* net, int32_t H, int32_t W, int32_t C, int32_t* out);
int rfx_net_conv(rfx_net* net, int32_t x, int32_t cout, int32_t R, int32_t S, int32_t stride, int32_t pad,
                 const char* name, int32_t* out);
/* convolution with rectangular padding (pad_h, pad_w); stride 1 unless square */
int rfx_net_conv2(rfx_net* net, int32_t x, int32_t cout, int32_t R, int32_t S, int32_t stride, int32_t pad_h,
                  int32_t pad_w, const char* name, int32_t* out);
int rfx_net_bn(rfx_net* net, int32_t y, int32_t relu, const char* name, int32_t* out);
int rfx_net_bn_add_relu(rfx_net* net, int32_t y, int32_t skip, const char* name, int32_t* out);
int rfx_net_relu(rfx_net* net, int32_t x, const char* name, int32_t* out);
int rfx_net_maxpool(rfx_net* net, int32_t x, int32_t k, int32_t stride, int32_t pad, const char* name,
                    int32_t* out);
int rfx_net_avgpool(rfx_net* net, int32_t x, const char* name, int32_t* out);
/* windowed average pooling (torch AvgPool2d, count_include_pad) */
int rfx_net_avgpool2d(rfx_net* net, int32_t x, int32_t k, int32_t stride, int32_t pad, const char* name,
                      int32_t* out);
/* hidden fully connected layer: NHWC input flattened, bf16 output [N, out_features] + bias */
int rfx_net_linear(rfx_net* net, int32_t x, int32_t out_features, const char* name, int32_t* out);
int rfx_net_fc(rfx_net* net, int32_t x, int32_t classes, const char* name, int32_t* out);
int rfx_net_concat(rfx_net* net, int32_t a, int32_t b, const char* name, int32_t* out);
int rfx_net_loss(rfx_net* net, int32_t logits, const char* name, int32_t* out);

/* introspection */
int32_t rfx_net_num_tensors(const rfx_net* net);
int rfx_net_tensor_info(const rfx_net* net, int32_t t, char* name, size_t name_cap, int32_t* nhwc,
                        int32_t* dtype, int64_t* cost, int32_t* producer);
int32_t rfx_net_num_ops(const rfx_net* net);
int rfx_net_op_info(const rfx_net* net, int32_t op, char* name, size_t name_cap, int32_t* kind,
                    int32_t* inputs /* up to 2, -1 pads */, int32_t* out);
/* attrs[8] = {R, S, stride, pad, k (pool window / bn relu flag), classes, cin_real, cout} */
/* attrs[9] = {R, S, stride, pad_h, k, classes, cin_real, cout, pad_w} */
int rfx_net_op_attrs(const rfx_net* net, int32_t op, int32_t* attrs);
int64_t rfx_net_flops_per_step(const rfx_net* net);

/* planning: policy "reforward" | "store_all" | "lcg" | "sqrt" */
int rfx_net_plan(rfx_net* net, const char* policy);
int rfx_net_plan_with_stored(rfx_net* net, const uint8_t* stored_mask, const char* label);

typedef struct rfx_memory_report {
  int64_t planned_total;     /* Eq. 1 of the plan: stored cost + largest segment */
  int64_t stored_cost;
  int64_t max_segment;
  int64_t store_all_total;   /* sum of interior tensor costs (regular training) */
  int64_t tracked_peak;      /* live activation high-water mark over the schedule */
  int64_t arena_bytes;       /* activation arena capacity */
  int64_t grad_arena_bytes;
  int64_t workspace_bytes;
  int64_t param_bytes;
  int64_t state_bytes;
  int64_t reforward_ops;
  int64_t segment_loads;
  int64_t forward_ops;
  int64_t backward_ops;
  int64_t launches_per_step; /* kernel nodes in the captured step graph (0 before capture) */
  int64_t candidate_max_term;
  int32_t n_segments;
  int32_t n_stored;
  int64_t device_bytes;      /* every device allocation of the net after setup (arena + guard band,
                                gradient arena, workspace, parameters / gradients / momentum, bf16
                                copies, BN state, input, staging, tables) */
} rfx_memory_report;

int rfx_net_plan_info(const rfx_net* net, uint8_t* stored_mask, int32_t* seg_of, rfx_memory_report* rep);
/* schedule: kinds (0 forward, 1 backward, 2 release), op ids, segment ids, re-forward flags,
 * phases (0 whole op; 1/2 = the two halves of a join whose inputs sit in two segments) */
int rfx_net_schedule(const rfx_net* net, int32_t* kinds, int32_t* ops, int32_t* segs, int32_t* reforward,
                     int32_t* phases, int32_t cap, int32_t* n_out);

/* runtime */
int rfx_net_setup(rfx_net* net, uint64_t seed);
/* images: NCHW fp32 [batch, C, H, W]; labels int32 [batch]; from_host: 1 host
 * pointers (copied inside the call), 0 device pointers */
/* Double-buffered input pipeline (slot 0/1): stage_batch copies a host batch
 * (pinned for overlap) to the slot on copy_stream once the slot's previous
 * batch was consumed; use_batch makes `stream` wait for it, packs it into the
 * network input and frees the slot.  Stage batch k+1 while step k runs. */
int rfx_net_stage_batch(rfx_net* net, const float* images_host, const int32_t* labels_host, int32_t slot,
                        void* copy_stream);
int rfx_net_use_batch(rfx_net* net, int32_t slot, void* stream);
int rfx_net_load_batch(rfx_net* net, const float* images, const int32_t* labels, int32_t from_host,
                       void* stream);
int rfx_net_forward_backward(rfx_net* net, void* stream);
int rfx_net_update(rfx_net* net, float lr, float momentum, float weight_decay, void* stream);
int rfx_net_step(rfx_net* net, float lr, float momentum, float weight_decay, int32_t use_graph, void* stream);
/* phase 0 forward+backward, 1 SGD update + weight prep, 2 both; with use_graph
 * each phase is captured once into a CUDA graph and replayed */
int rfx_net_run_phase(rfx_net* net, int32_t phase, float lr, float momentum, float weight_decay,
                      int32_t use_graph, void* stream);
int rfx_net_read_loss(rfx_net* net, float* loss, void* stream);
/* enqueue the D2H copy of the step's loss into host_dst (pinned memory: no
 * host synchronisation; the value is valid once the stream reaches it) */
int rfx_net_copy_loss(rfx_net* net, float* host_dst, void* stream);
/* live roofline probe: replay exactly the step's GEMM launches; ms and
 * algorithmic flops per step, number of GEMM launches */
int rfx_net_gemm_profile(rfx_net* net, int32_t iters, void* stream, double* ms_per_step,
                         double* flops_per_step, int64_t* launches);
/* per GEMM launch of the step: 10 doubles {M, N, K, a_kind, b_kind, splits, ms, flops,
 * algorithmic bytes, tile width BLOCK_N} */
int rfx_net_gemm_profile_detail(rfx_net* net, int32_t iters, void* stream, double* rows, int32_t cap,
                                int32_t* n_out);

/* in-stream ms of every schedule instruction (eager launches, events between
 * them, mean over iters) and of the SGD update last: |schedule| + 1 doubles.
 * Runs forward/backward for real; the update uses lr 0. */
int rfx_net_instr_profile(rfx_net* net, int32_t iters, void* stream, double* ms, int32_t cap, int32_t* n_out);

/* tuning probe: ms of traced GEMM `idx` re-launched with a forced tile width
 * (64/128/256) and split-K count, writing fp32 partials to a scratch buffer */
int rfx_net_gemm_try(rfx_net* net, int32_t idx, int32_t block_n, int32_t splits, int32_t iters, void* stream,
                     double* ms);

/* 1 when no kernel wrote past the activation arena (sized to the planner's
 * Eq. 1 total): a canary band behind it is checked */
int rfx_net_arena_guard(const rfx_net* net, int32_t* intact);

int32_t rfx_net_num_params(const rfx_net* net);
int rfx_net_param_info(const rfx_net* net, int32_t i, char* name, size_t name_cap, int32_t* shape,
                       int32_t* ndim, int32_t* kind, int64_t* count);
/* which: 0 value, 1 gradient, 2 momentum; canonical (PyTorch OIHW / [out,in] / [C]) layout */
int rfx_net_read_param(const rfx_net* net, int32_t i, int32_t which, float* host);
int rfx_net_write_param(rfx_net* net, int32_t i, const float* host);
/* Host-only layout of the flat fp32 parameter / gradient buffers (what the
 * data-parallel all-reduce buckets cover): parameter i occupies
 * [offset, offset + count); pack writes a canonical tensor into that slice's
 * layout (padding zeroed), unpack reads it back.  No device access. */
int rfx_net_param_slot(const rfx_net* net, int32_t i, int64_t* offset, int64_t* count);
int rfx_net_pack_param(const rfx_net* net, int32_t i, const float* canonical, float* flat_slice);
int rfx_net_unpack_param(const rfx_net* net, int32_t i, const float* flat_slice, float* canonical);
int rfx_net_read_tensor(const rfx_net* net, int32_t t, float* host); /* NHWC, valid if resident */
int rfx_net_read_bn_running(const rfx_net* net, int32_t op, float* mean, float* var);
/* debug: give every activation gradient its own slot (call before plan) and read it back */
int rfx_net_set_keep_grads(rfx_net* net, int32_t on);
int rfx_net_read_grad_tensor(const rfx_net* net, int32_t t, float* host);
/* flat fp32 gradient buffer (data-parallel all-reduce target) */
int rfx_net_grad_buffer(const rfx_net* net, void** dev_ptr, int64_t* count);

/* data parallel over NCCL: rank 0 creates the 128-byte unique id, every rank
 * passes it to rfx_net_set_comm (after setup); the step then averages the
 * gradient buffer bucket by bucket on a side stream as the backward finishes
 * each range (overlapped, captured in the step graph) */
int rfx_comm_unique_id(char* id128);
int rfx_net_set_comm(rfx_net* net, int32_t nranks, int32_t rank, const char* id128, int64_t bucket_bytes);
int32_t rfx_net_comm_buckets(const rfx_net* net);
/* dry run of the bucket plan (no GPU needed): per bucket, the schedule
 * instruction after which it is reduced and its float range [lo, hi) */
int rfx_net_bucket_plan(rfx_net* net, int64_t bucket_bytes, int32_t* after_instr, int64_t* lo, int64_t* hi,
                        int32_t cap, int32_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* REFORWARD_B200_EXEC_H_ */
