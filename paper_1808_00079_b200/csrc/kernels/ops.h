// Launchers of the non-GEMM kernels (csrc/kernels/ops.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace rfk {

struct PoolGeom {
  int N, H, W, C, P, Q, k, stride, pad;
};

struct ConvShape {  // for the explicit im2col path
  int N, H, W, C, Cs /*channel stride of x*/, P, Q, R, S, stride, pad;
};

int colstats_blocks(long M);
cudaError_t colstats(const __nv_bfloat16* x, long M, int C, float* partials, int blocks, cudaStream_t st);
cudaError_t bn_finalize(const float* partials, int parts, int C, long count, const float* gamma, const float* beta,
                        float eps, float* mean, float* invstd, float* scale, float* shift, float* run_mean,
                        float* run_var, float momentum, bool update_running, cudaStream_t st);
// BatchNorm over a channel concatenation: the statistics of every 32-channel
// block come from the partial-sum rows of the tensor that produced those
// channels (computed once per tensor, not once per consuming layer)
struct BnGatherBlock {
  const float* partials;  // [parts][2][Csrc]
  int parts, Csrc, coff;  // rows, source channels, channel offset of this block in the source
};
cudaError_t bn_finalize_gather(const BnGatherBlock* table, int C, long count, const float* gamma, const float* beta,
                               float eps, float* mean, float* invstd, float* scale, float* shift, float* run_mean,
                               float* run_var, float momentum, cudaStream_t st);
cudaError_t bn_apply(const __nv_bfloat16* y, const __nv_bfloat16* skip, const float* scale, const float* shift,
                     bool relu, long M, int C, __nv_bfloat16* out, cudaStream_t st);
// mask_mode: 0 none (plain BN), 1 relu(bn(y)), 2 relu via stored output (> 0)
cudaError_t bn_backward(const __nv_bfloat16* y, const __nv_bfloat16* dout, const __nv_bfloat16* out, int mask_mode,
                        const float* gamma, const float* mean, const float* invstd, const float* scale,
                        const float* shift, long M, int C, float* partials, int blocks, float* coef, float* dgamma,
                        float* dbeta, __nv_bfloat16* dy, bool acc_dy, __nv_bfloat16* dskip, bool acc_dskip,
                        cudaStream_t st);
// BN+ReLU backward from statistics rows [parts][2][C] of (sum g, sum g*(y-mean))
// (written by the consumer conv's dgrad epilogue or its replay): finalize,
// then dy (+)= k1*g + k2*y + k3 with g = dout * [y*scale + shift > 0]
cudaError_t bn_backward_from_rows(const __nv_bfloat16* y, const __nv_bfloat16* dout, const float* gamma,
                                  const float* mean, const float* invstd, const float* scale, const float* shift,
                                  long M, int C, const float* rows, int parts, float* coef, float* dgamma,
                                  float* dbeta, __nv_bfloat16* dy, bool acc_dy, cudaStream_t st);
cudaError_t relu_fwd(const __nv_bfloat16* x, long n, __nv_bfloat16* y, cudaStream_t st);
cudaError_t relu_bwd(const __nv_bfloat16* y, const __nv_bfloat16* dy, long n, __nv_bfloat16* dx, bool acc,
                     cudaStream_t st);
// idx (optional): first-argmax window position per output (k*k <= 256), read
// back by maxpool_bwd_from_idx (the backward then never re-reads x)
cudaError_t maxpool_fwd(const __nv_bfloat16* x, const PoolGeom& g, __nv_bfloat16* y, cudaStream_t st,
                        uint8_t* idx = nullptr);
cudaError_t maxpool_bwd_from_idx(const uint8_t* idx, const __nv_bfloat16* dy, const PoolGeom& g, __nv_bfloat16* dx,
                                 bool acc, cudaStream_t st);
// idx_ws: N*P*Q*C bytes of scratch (window argmax)
cudaError_t maxpool_bwd(const __nv_bfloat16* x, const __nv_bfloat16* y, const __nv_bfloat16* dy, const PoolGeom& g,
                        __nv_bfloat16* dx, bool acc, void* idx_ws, cudaStream_t st);
// windowed average pooling (count_include_pad) and its gather backward
cudaError_t avgpool2d_fwd(const __nv_bfloat16* x, const PoolGeom& g, __nv_bfloat16* y, cudaStream_t st);
cudaError_t avgpool2d_bwd(const __nv_bfloat16* dy, const PoolGeom& g, __nv_bfloat16* dx, bool acc, cudaStream_t st);
cudaError_t avgpool_fwd(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* out, cudaStream_t st);
cudaError_t avgpool_bwd(const __nv_bfloat16* dout, int N, int HW, int C, __nv_bfloat16* dx, bool acc,
                        cudaStream_t st);
cudaError_t softmax_ce_fwd(const float* logits, const int* labels, int N, int K, float* row_loss, float* lse,
                           float* loss, cudaStream_t st);
cudaError_t softmax_ce_bwd(const float* logits, const int* labels, const float* lse, int N, int K, float* dlogits,
                           cudaStream_t st);
cudaError_t cast_f32_bf16(const float* x, long n, __nv_bfloat16* y, cudaStream_t st);
// n % 8 == 0, 16-byte aligned buffers: 8 elements per thread-iteration
cudaError_t cast_f32_bf16_vec(const float* x, long n, __nv_bfloat16* y, cudaStream_t st);
cudaError_t cast_f32_bf16_2d(const float* x, int R, int C, int ldo, __nv_bfloat16* y, cudaStream_t st);
cudaError_t colsum_bf16(const __nv_bfloat16* x, int R, int C, float* out, bool acc, cudaStream_t st);
cudaError_t colsum_f32(const float* x, int R, int C, float* out, bool acc, cudaStream_t st);
// split-K finish into a bf16 activation ([M][N] rows, stride ldc), optional
// BN statistics rows (<= max_blocks rows of [2][N], the conv's stats slot)
cudaError_t reduce_splits_bf16(const float* parts, int splits, int M, int N, __nv_bfloat16* out, long ldc, bool acc,
                               float* stats, int max_blocks, cudaStream_t st);
cudaError_t reduce_splits(const float* parts, int splits, long n, float* out, bool acc, cudaStream_t st);
// hyper: device {lr, momentum, weight decay}; wb (optional): bf16 copy of w
// refreshed in the same pass
cudaError_t sgd_update(float* w, const float* g, float* m, long n, const float* hyper, __nv_bfloat16* wb,
                       cudaStream_t st);
cudaError_t conv_weight_prep(const float* w, int Cout, int R, int S, int Cpad, int Cin, int CoutPad,
                             __nv_bfloat16* wb, __nv_bfloat16* wt, cudaStream_t st);
// One launch for every conv / fc layer after an SGD step: bf16 copy of the
// GEMM-layout weights plus (convs) the flipped transpose used by dgrad.  The
// table lives in device memory; `starts` are element offsets of each layer
// in the virtual concatenation [copy elems | transpose elems].
struct WeightPrepLayer {
  const float* w;
  __nv_bfloat16* wb;
  __nv_bfloat16* wt;  // nullptr: no transpose
  int cout, R, S, cpad, cin, coutpad;
  long n_copy, n_t;   // elements of wb and of wt
  long start;         // first virtual element of this layer
};
cudaError_t weight_prep_batched(const WeightPrepLayer* table_dev, int layers, long total, cudaStream_t st);
cudaError_t pack_input(const float* x, int N, int C, int H, int W, int Cpad, __nv_bfloat16* out, cudaStream_t st);
cudaError_t im2col(const __nv_bfloat16* x, const ConvShape& g, int Kpad, __nv_bfloat16* out, cudaStream_t st);
// zero fill / device copy as PDL kernels (16-byte aligned; else cudaMemset / cudaMemcpy)
cudaError_t fill_zero(void* p, long bytes, cudaStream_t st);
cudaError_t copy_bytes(void* dst, const void* src, long bytes, cudaStream_t st);
cudaError_t zero_insert(const __nv_bfloat16* dy, int N, int P, int Q, int C, int Hu, int Wu, int stride,
                        __nv_bfloat16* u, cudaStream_t st);
cudaError_t concat(const __nv_bfloat16* a, int Ca, const __nv_bfloat16* b, int Cb, long M, __nv_bfloat16* c,
                   cudaStream_t st);
cudaError_t split_grad(const __nv_bfloat16* dc, int Ca, int Cb, long M, __nv_bfloat16* da, bool acc_a,
                       __nv_bfloat16* db, bool acc_b, cudaStream_t st);
cudaError_t add_bf16(const __nv_bfloat16* a, long n, __nv_bfloat16* dst, cudaStream_t st);

}  // namespace rfk
