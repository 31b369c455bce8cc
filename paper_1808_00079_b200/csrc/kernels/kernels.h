// Host-side interface of the sm_100a kernels (internal; the C-ABI wrappers
// live in csrc/executor/exec_capi.cpp).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace rfk {

// ------------------------------------------------------------ GEMM engine
// One warp-specialised tcgen05 kernel family serves every dense contraction of
// the train step: conv fprop / dgrad (implicit GEMM through TMA im2col), conv
// wgrad (im2col operand in MN-major form), 1x1 convs and the classifier (plain
// 2-D TMA).  D[M,N] = sum_k A[m,k] * B[n,k], bf16 operands, fp32 accumulate in
// TMEM.
enum class Operand : int {
  KMajor2D = 0,   // rows x K, K contiguous (row stride `ld` elements)
  MNMajor2D = 1,  // K rows x MN, MN contiguous (row stride `ld` elements)
  Im2colK = 2,    // NHWC activation, rows = output pixels, K = (r, s, c)
  Im2colMN = 3,   // NHWC activation, K = output pixels, MN = (r, s, c)
  // conv weights [Cout][R][S][Cpad] read as the dgrad B operand: MN = input
  // channel (contiguous), K = (flipped tap, Cout) — no transposed copy needed
  WeightTapsMN = 4,
};

// Convolution geometry for an im2col operand: input tensor N x H x W x C,
// output P x Q, filter R x S.  c_blocks = ceil(C / 64); the K (or MN) index of
// tap (r, s) channel c is ((r * S + s) * c_blocks * 64 + c).
struct ConvGeom {
  int N = 0, H = 0, W = 0, C = 0;
  int P = 0, Q = 0, R = 1, S = 1;
  int pad_h = 0, pad_w = 0, stride_h = 1, stride_w = 1;
};

struct GemmDesc {
  int M = 0, N = 0, K = 0;
  Operand a_kind = Operand::KMajor2D;
  const void* a = nullptr;
  long a_ld = 0;
  ConvGeom a_geom;
  Operand b_kind = Operand::KMajor2D;
  const void* b = nullptr;
  long b_ld = 0;
  ConvGeom b_geom;
  long b_extent = 0;  // valid MN extent of an MN-major B (0 = N)
  int b_taps = 1, b_cpad = 0, b_rows = 0;  // WeightTapsMN: R*S, Cpad, Cout
  // WeightTapsMN: weight tap read for A tap (r, s) = base - r * dr - s * ds
  // (base < 0: the flipped full filter, R*S - 1 - tap)
  int b_tap_base = -1, b_tap_dr = 0, b_tap_ds = 0;
  // epilogue
  void* out = nullptr;
  long ldc = 0;
  bool out_f32 = false;
  bool accumulate_out = false;  // out += D (fp32 or bf16)
  const float* bias = nullptr;  // per column
  float* stats = nullptr;       // [m_tiles][2][N] column sum / sum of squares
  bool stats_acc = false;       // add to the statistics rows instead of writing them (chunked M)
  int splits = 1;               // split-K; split z writes out + z * split_stride
  long split_stride = 0;
  // row remap of the output (strided-conv dgrad scatter): row m = (n, p, q)
  // over P x Q goes to n * H * W + (p * sh) * W + q * sw.
  bool remap = false;
  int rP = 0, rQ = 0, rH = 0, rW = 0, rsh = 1, rsw = 1;
  int block_n = 0;  // 0 = pick automatically (64 / 128 / 256)
  // Im2colK A of a stride-1 conv: the shifted-band kernel (gemm_band.cu).
  // 0 never; 1 where gemm_band_preferred() (measured faster than TMA im2col);
  // 2 wherever gemm_band_ok() accepts the shape
  int band = 0;
  // fused BatchNorm apply on the bf16 output (re-forward, statistics known):
  // bn_out = [relu](out * bn_scale + bn_shift), per column
  void* bn_out = nullptr;
  const float* bn_scale = nullptr;
  const float* bn_shift = nullptr;
  bool bn_relu = false;
  // persistent grid cap (0 = one CTA per SM): leaves SMs free for NCCL kernels
  // on a side stream while gradient buckets are in flight
  int max_ctas = 0;
  // BN backward statistics (with `stats`, bf16 output = dout of a BN+ReLU
  // output, stored as is): rows of (sum g, sum g * (bs_y - bs_mean)) per
  // column, g = dout * [bs_y * bs_scale + bs_shift > 0], instead of (sum, sum^2).
  // replay: no GEMM; the epilogue re-reads `out` and emits the same rows a
  // fused launch of the same M / N / block_n would (bit-identical).
  bool stats_bwd = false;
  bool replay = false;
  const void* bs_y = nullptr;  // bf16 [M][bs_ldy]: the BN input
  long bs_ldy = 0;
  const float* bs_mean = nullptr;
  const float* bs_scale = nullptr;
  const float* bs_shift = nullptr;
  // CTA pairs (2-CTA clusters, cta_group::2 M = 256 tiles): 0 = automatic
  // (long plain-operand main loops), 1 = wherever the shapes allow, -1 = never
  int pair = 0;
};

cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t stream);
bool gemm_band_ok(const GemmDesc& d);
bool gemm_band_preferred(const GemmDesc& d);
cudaError_t gemm_band_launch(const GemmDesc& d, cudaStream_t stream);
int gemm_m_tiles(const GemmDesc& d);
int gemm_block_n(const GemmDesc& d);  // tile width the launch will use

}  // namespace rfk
