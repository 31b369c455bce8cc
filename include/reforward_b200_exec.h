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
} rfx_gemm_args;

int rfx_gemm(const rfx_gemm_args* args, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* REFORWARD_B200_EXEC_H_ */
