// rfx_* kernel-level C-ABI entry points (include/reforward_b200_exec.h).
#include <cuda_runtime.h>

#include <string>

#include "kernels/kernels.h"
#include "kernels/ops.h"
#include "reforward_b200.h"

namespace rfexec {
void set_last_error(const std::string& msg);
}

namespace {
rfk::ConvGeom to_geom(const rfx_conv_geom& g) {
  rfk::ConvGeom o;
  o.N = g.N; o.H = g.H; o.W = g.W; o.C = g.C; o.P = g.P; o.Q = g.Q; o.R = g.R; o.S = g.S;
  o.pad_h = g.pad_h; o.pad_w = g.pad_w; o.stride_h = g.stride_h; o.stride_w = g.stride_w;
  return o;
}
}  // namespace

extern "C" size_t rfx_gemm_args_size(void) { return sizeof(rfx_gemm_args); }

extern "C" int rfx_gemm(const rfx_gemm_args* a, void* stream) {
  rfk::GemmDesc d;
  d.M = a->M; d.N = a->N; d.K = a->K;
  d.a_kind = static_cast<rfk::Operand>(a->a_kind); d.a = a->a; d.a_ld = a->a_ld; d.a_geom = to_geom(a->a_geom);
  d.b_kind = static_cast<rfk::Operand>(a->b_kind); d.b = a->b; d.b_ld = a->b_ld; d.b_geom = to_geom(a->b_geom);
  d.out = a->out; d.ldc = a->ldc; d.out_f32 = a->out_f32 != 0; d.accumulate_out = a->accumulate_out != 0;
  d.bias = a->bias; d.stats = a->stats; d.splits = a->splits; d.split_stride = a->split_stride;
  d.remap = a->remap != 0; d.rP = a->rP; d.rQ = a->rQ; d.rH = a->rH; d.rW = a->rW; d.rsh = a->rsh; d.rsw = a->rsw;
  d.block_n = a->block_n;
  d.b_extent = a->b_extent;
  d.b_taps = a->b_taps > 0 ? a->b_taps : 1;
  d.b_cpad = a->b_cpad;
  d.b_rows = a->b_rows;
  d.band = a->band != 0 ? 2 : 0;  // the C-ABI flag forces the band kernel where the shape allows it
  if (a->b_tap_map) {
    d.b_tap_base = a->b_tap_base;
    d.b_tap_dr = a->b_tap_dr;
    d.b_tap_ds = a->b_tap_ds;
  }
  d.stats_bwd = a->stats_bwd != 0;
  d.replay = a->replay != 0;
  d.bs_y = a->bs_y;
  d.bs_ldy = a->bs_ldy;
  d.bs_mean = a->bs_mean;
  d.bs_scale = a->bs_scale;
  d.bs_shift = a->bs_shift;
  d.pair = a->pair;
  cudaError_t e = rfk::gemm_launch(d, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    rfexec::set_last_error(std::string("rfx_gemm: ") + cudaGetErrorString(e));
    return RF_E_CUDA;
  }
  return RF_OK;
}

extern "C" int rfx_im2col(const void* x, int N, int H, int W, int C, int Cs, int P, int Q, int R, int S, int stride,
                          int pad, int kpad, void* out, void* stream) {
  rfk::ConvShape g{N, H, W, C, Cs, P, Q, R, S, stride, pad};
  cudaError_t e = rfk::im2col(static_cast<const __nv_bfloat16*>(x), g, kpad, static_cast<__nv_bfloat16*>(out),
                              static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    rfexec::set_last_error(std::string("rfx_im2col: ") + cudaGetErrorString(e));
    return RF_E_CUDA;
  }
  return RF_OK;
}

extern "C" int rfx_maxpool_bwd(const void* x, const void* dy, int N, int H, int W, int C, int k, int stride, int pad,
                               void* dx, int accumulate, void* workspace, void* stream) {
  rfk::PoolGeom g{N, H, W, C, (H + 2 * pad - k) / stride + 1, (W + 2 * pad - k) / stride + 1, k, stride, pad};
  cudaError_t e = rfk::maxpool_bwd(static_cast<const __nv_bfloat16*>(x), nullptr, static_cast<const __nv_bfloat16*>(dy),
                                   g, static_cast<__nv_bfloat16*>(dx), accumulate != 0, workspace,
                                   static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    rfexec::set_last_error(std::string("rfx_maxpool_bwd: ") + cudaGetErrorString(e));
    return RF_E_CUDA;
  }
  return RF_OK;
}
