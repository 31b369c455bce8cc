// HBM-streaming kernels of the train step (everything that is not a dense
// contraction): BatchNorm statistics / apply / backward, ReLU, pooling,
// softmax cross-entropy, SGD, weight layout transforms, input packing.
//
// All activations are NHWC bf16 with C % 8 == 0, so one 16-byte vector is 8
// consecutive channels of one pixel.  Every reduction is a fixed-shape tree
// (no atomics): results are bit-reproducible run to run, which is what makes
// re-forward gradients bit-identical to store-all gradients.
#include <cstdlib>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>

#include "kernels/launch.cuh"
#include "kernels/ops.h"

namespace rfk {

#define RFK_CHECK_LAUNCH(call)            \
  do {                                    \
    const cudaError_t e_ = (call);        \
    if (e_ != cudaSuccess) return e_;     \
  } while (0)

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

__device__ __forceinline__ uint4 ldg16(const void* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

__device__ __forceinline__ uint32_t pack_bf16_pair(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

int grid_for(long work, int per_block, int cap = 148 * 16) {
  long g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

// ------------------------------------------------------------ column reductions
// Layout of a reduction launch over an [M, C] bf16 matrix: a block owns a
// contiguous slab of rows; its threads are arranged as (rows_per_pass x tpr)
// with tpr = C / 8 vector lanes per row.  Each thread accumulates its 8
// channels over its rows; threads sharing channels are then summed in smem in
// a fixed order and the block writes partials[block][2][C].
struct RedShape {
  int tpr;            // threads per row (C / 8), <= 256
  int rows_per_pass;  // 256 / tpr
};

__device__ __forceinline__ RedShape red_shape(int C) {
  RedShape s;
  s.tpr = C / 8;
  s.rows_per_pass = kThreads / s.tpr;
  return s;
}

// mode: 0 = plain column sum / sum of squares of x
template <int MODE>
__global__ void __launch_bounds__(kThreads) colstats_kernel(const __nv_bfloat16* __restrict__ x, long M, int C,
                                                            long rows_per_block, float* __restrict__ partials, int cw) {
  pdl_enter();
  // handles cw <= 2048 channels per pass; channel chunks via blockIdx.y
  __shared__ float sh[2][kThreads][8];
  const int cchunk = blockIdx.y;  // chunk of cw channels
  const int Cc = min(cw, C - cchunk * cw);
  const RedShape s = red_shape(Cc);
  const int t = threadIdx.x;
  const int lane = t % s.tpr, rgrp = t / s.tpr;
  float a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = b[i] = 0.f;
  const long r0 = (long)blockIdx.x * rows_per_block;
  const long r1 = min(M, r0 + rows_per_block);
  if (rgrp < s.rows_per_pass) {
    for (long r = r0 + rgrp; r < r1; r += s.rows_per_pass) {
      float f[8];
      unpack8(ldg16(x + r * C + cchunk * cw + lane * 8), f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] += f[i];
        b[i] += f[i] * f[i];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    sh[0][t][i] = a[i];
    sh[1][t][i] = b[i];
  }
  __syncthreads();
  if (t < s.tpr) {
    for (int g = 1; g < s.rows_per_pass; ++g)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] += sh[0][g * s.tpr + t][i];
        b[i] += sh[1][g * s.tpr + t][i];
      }
    float* out = partials + (long)blockIdx.x * 2 * C + cchunk * cw + t * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      out[i] = a[i];
      out[C + i] = b[i];
    }
  }
}

// Sum `parts` partial rows [parts][2][C] in a fixed tree: channel per
// threadIdx.x (32 wide), partial subsets per threadIdx.y (32 deep, two
// independent accumulators each), then a fixed butterfly over the subsets.
// The sums of channel blockIdx.x * 32 + j are returned to warp j (threadIdx.y
// == j; the caller's channel is fin_channel()).
constexpr int kFinY = 32;
__device__ __forceinline__ int fin_channel() { return blockIdx.x * 32 + threadIdx.y; }
__device__ __forceinline__ void sum_partials(const float* __restrict__ partials, int parts, int C, int c, float& s0,
                                             float& s1) {
  __shared__ float sh0[kFinY][33], sh1[kFinY][33];
  float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
  if (c < C) {
    // rows y + 32k: even k into (a0, b0), odd k into (a1, b1), ascending k.
    // Eight rows' loads are issued before any add (the finalize is one
    // L2 round trip per batch, not per row); the add order is unchanged.
    for (int k0 = 0; (int)threadIdx.y + kFinY * k0 < parts; k0 += 8) {
      float va[8], vb[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int p = (int)threadIdx.y + kFinY * (k0 + j);
        va[j] = p < parts ? __ldg(partials + (long)p * 2 * C + c) : 0.f;
        vb[j] = p < parts ? __ldg(partials + (long)p * 2 * C + C + c) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if ((int)threadIdx.y + kFinY * (k0 + j) >= parts) break;
        if (j & 1) {
          a1 += va[j];
          b1 += vb[j];
        } else {
          a0 += va[j];
          b0 += vb[j];
        }
      }
    }
  }
  sh0[threadIdx.y][threadIdx.x] = a0 + a1;
  sh1[threadIdx.y][threadIdx.x] = b0 + b1;
  __syncthreads();
  // transposed: warp y reduces channel y's 32 row-group sums (lane = row
  // group) with a fixed xor butterfly -- one barrier instead of a 5-level
  // smem tree with a barrier per level.  The results land in warp y (every
  // lane) for channel blockIdx.x * 32 + y.
  float t0 = sh0[threadIdx.x][threadIdx.y], t1 = sh1[threadIdx.x][threadIdx.y];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    t0 += __shfl_xor_sync(0xffffffffu, t0, off);
    t1 += __shfl_xor_sync(0xffffffffu, t1, off);
  }
  s0 = t0;
  s1 = t1;
}

__global__ void bn_finalize_kernel(const float* __restrict__ partials, int parts, int C, float count,
                                   const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                                   float* __restrict__ mean, float* __restrict__ invstd, float* __restrict__ scale,
                                   float* __restrict__ shift, float* __restrict__ run_mean, float* __restrict__ run_var,
                                   float momentum, int update_running) {
  pdl_enter();
  float s0, s1;
  sum_partials(partials, parts, C, blockIdx.x * 32 + threadIdx.x, s0, s1);
  const int c = fin_channel();
  if (threadIdx.x != 0 || c >= C) return;
  const float mu = s0 / count;
  const float var = fmaxf(s1 / count - mu * mu, 0.f);
  const float is = rsqrtf(var + eps);
  mean[c] = mu;
  invstd[c] = is;
  const float sc = gamma[c] * is;
  scale[c] = sc;
  shift[c] = beta[c] - mu * sc;
  if (update_running) {
    const float unbiased = count > 1.f ? var * count / (count - 1.f) : var;
    run_mean[c] = (1.f - momentum) * run_mean[c] + momentum * mu;
    run_var[c] = (1.f - momentum) * run_var[c] + momentum * unbiased;
  }
}

// Finalize of a BN over a concatenation: block b takes its 32 channels' sums
// from the rows of their source tensor (table[b]).
__global__ void bn_finalize_gather_kernel(const BnGatherBlock* __restrict__ table, int C, float count,
                                          const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
                                          float* __restrict__ mean, float* __restrict__ invstd,
                                          float* __restrict__ scale, float* __restrict__ shift,
                                          float* __restrict__ run_mean, float* __restrict__ run_var, float momentum) {
  pdl_enter();
  const BnGatherBlock b = table[blockIdx.x];
  float s0, s1;
  sum_partials(b.partials, b.parts, b.Csrc, b.coff + (int)threadIdx.x, s0, s1);
  const int c = fin_channel();
  if (threadIdx.x != 0 || c >= C) return;
  const float mu = s0 / count;
  const float var = fmaxf(s1 / count - mu * mu, 0.f);
  const float is = rsqrtf(var + eps);
  mean[c] = mu;
  invstd[c] = is;
  const float sc = gamma[c] * is;
  scale[c] = sc;
  shift[c] = beta[c] - mu * sc;
  const float unbiased = count > 1.f ? var * count / (count - 1.f) : var;
  run_mean[c] = (1.f - momentum) * run_mean[c] + momentum * mu;
  run_var[c] = (1.f - momentum) * run_var[c] + momentum * unbiased;
}

// out = [relu](y * scale + shift [+ skip])
// (skip may alias out: each element is read before it is written)
__device__ __forceinline__ void ld8f(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
  f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
}

// Each thread streams kVec 16-byte vectors per iteration, all loads issued
// before any math, so every SM keeps enough bytes in flight for HBM.
// Four 16-byte vectors per thread in flight (plus the skip operand), 32-bit
// indexing, SKIP / RELU resolved at compile time.
constexpr int kVec = 4;

template <bool SKIP, bool RELU>
__global__ void __launch_bounds__(kThreads) bn_apply_kernel(const __nv_bfloat16* __restrict__ y,
                                                           const __nv_bfloat16* skip, const float* __restrict__ scale,
                                                           const float* __restrict__ shift, unsigned nvec, int C,
                                                           __nv_bfloat16* out) {
  pdl_enter();
  const unsigned cv = (unsigned)C / 8;
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < nvec; v0 += stride * kVec) {
    uint4 yv[kVec], kv[kVec];
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const unsigned v = v0 + u * stride;
      if (v < nvec) {
        yv[u] = ldg16(y + (size_t)v * 8);
        if (SKIP) kv[u] = *reinterpret_cast<const uint4*>(skip + (size_t)v * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < kVec; ++u) {
      const unsigned v = v0 + u * stride;
      if (v >= nvec) break;
      const int c0 = (int)(v % cv) * 8;
      float f[8], sc[8], sh[8];
      unpack8(yv[u], f);
      ld8f(scale + c0, sc);
      ld8f(shift + c0, sh);
      if (SKIP) {
        float k[8];
        unpack8(kv[u], k);
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], sc[i], sh[i]) + k[i];
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fmaf(f[i], sc[i], sh[i]);
      }
      if (RELU) {
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fmaxf(f[i], 0.f);
      }
      *reinterpret_cast<uint4*>(out + (size_t)v * 8) = pack8(f);
    }
  }
}

// Backward reduction: g = dout * mask, accumulate sum(g) and sum(g * (y - mean))
// (the finalize scales the second sum by invstd, so the inner loop carries
// only the mean).  MODE: 0 no mask, 1 relu recomputed from y*scale+shift
// (same expression as the forward), 2 relu of the stored output (out > 0).
// Two rows per thread in flight and <= 85 registers (3 blocks of 256 per SM)
// keep enough loads outstanding for HBM.
// gout (MODE 2 only, optional): also store g = dout * mask -- the residual
// add's skip gradient -- so the apply pass reads g instead of dout and out.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 3) bn_bwd_reduce_kernel(
    const __nv_bfloat16* __restrict__ y, const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
    const float* __restrict__ mean, const float* __restrict__ scale, const float* __restrict__ shift, long M, int C,
    long rows_per_block, float* __restrict__ partials, __nv_bfloat16* __restrict__ gout, int cw) {
  pdl_enter();
  __shared__ float sh[2][kThreads][8];
  const int cchunk = blockIdx.y;
  const int Cc = min(cw, C - cchunk * cw);
  const RedShape s = red_shape(Cc);
  const int t = threadIdx.x;
  const int lane = t % s.tpr, rgrp = t / s.tpr;
  const int c0 = cchunk * cw + lane * 8;
  float a[8], b[8], mu[8], sc[8], sf[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = b[i] = 0.f;
  const long r0 = (long)blockIdx.x * rows_per_block;
  const long r1 = min(M, r0 + rows_per_block);
  if (rgrp < s.rows_per_pass) {
    ld8f(mean + c0, mu);
    if (MODE == 1) {
      ld8f(scale + c0, sc);
      ld8f(shift + c0, sf);
    }
    const long step = s.rows_per_pass;
    for (long r = r0 + rgrp; r < r1; r += 2 * step) {
      const bool two = r + step < r1;
      const long off0 = r * C + c0, off1 = (r + step) * C + c0;
      uint4 uy[2], ud[2], uo[2];
      uy[0] = ldg16(y + off0);
      ud[0] = ldg16(dout + off0);
      if (MODE == 2) uo[0] = ldg16(out + off0);
      if (two) {
        uy[1] = ldg16(y + off1);
        ud[1] = ldg16(dout + off1);
        if (MODE == 2) uo[1] = ldg16(out + off1);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && !two) break;
        float fy[8], fd[8], fo[8];
        unpack8(uy[u], fy);
        unpack8(ud[u], fd);
        if (MODE == 2) unpack8(uo[u], fo);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float g = fd[i];
          if (MODE == 1) g = (fmaf(fy[i], sc[i], sf[i]) > 0.f) ? g : 0.f;
          if (MODE == 2) g = (fo[i] > 0.f) ? g : 0.f;
          fd[i] = g;
          a[i] += g;
          b[i] = fmaf(g, fy[i] - mu[i], b[i]);
        }
        // g is dout with some lanes zeroed: exactly representable, so the
        // stored bf16 equals what the separate apply pass would write
        if (MODE == 2 && gout) *reinterpret_cast<uint4*>(gout + (u ? off1 : off0)) = pack8(fd);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    sh[0][t][i] = a[i];
    sh[1][t][i] = b[i];
  }
  __syncthreads();
  if (t < s.tpr) {
    for (int gi = 1; gi < s.rows_per_pass; ++gi)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] += sh[0][gi * s.tpr + t][i];
        b[i] += sh[1][gi * s.tpr + t][i];
      }
    float* o = partials + (long)blockIdx.x * 2 * C + cchunk * cw + t * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i] = a[i];
      o[C + i] = b[i];
    }
  }
}

// dbeta = sum g, dgamma = invstd * sum g*(y-mean); dy = k1*g + k2*y + k3
__global__ void bn_bwd_finalize_kernel(const float* __restrict__ partials, int parts, int C, float count,
                                       const float* __restrict__ gamma, const float* __restrict__ mean,
                                       const float* __restrict__ invstd, float* __restrict__ dgamma,
                                       float* __restrict__ dbeta, float* __restrict__ coef) {
  pdl_enter();
  float sg, sgy;
  sum_partials(partials, parts, C, blockIdx.x * 32 + threadIdx.x, sg, sgy);
  const int c = fin_channel();
  if (threadIdx.x != 0 || c >= C) return;
  const float is = invstd[c];
  const float sgx = sgy * is;
  dbeta[c] = sg;
  dgamma[c] = sgx;
  const float k1 = gamma[c] * is;
  const float k2 = -k1 * is * sgx / count;
  const float k3 = -k1 * sg / count - k2 * mean[c];
  coef[c] = k1;
  coef[C + c] = k2;
  coef[2 * C + c] = k3;
}

// dy (+)= k1*g + k2*y + k3 with g = dout * mask; dskip (+)= g (residual add).
// Two vectors per thread in flight; <= 64 registers.
template <int MODE, bool SKIP>
__global__ void __launch_bounds__(kThreads, 4) bn_bwd_apply_kernel(
    const __nv_bfloat16* __restrict__ y, const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ out,
    const float* __restrict__ scale, const float* __restrict__ shift, const float* __restrict__ coef, unsigned nvec,
    int C, __nv_bfloat16* __restrict__ dy, int acc_dy, __nv_bfloat16* __restrict__ dskip, int acc_dskip) {
  pdl_enter();
  const unsigned cv = (unsigned)C / 8;
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < nvec; v0 += 2 * stride) {
    uint4 uy[2], ud[2], uo[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const unsigned v = v0 + u * stride;
      if (v < nvec) {
        uy[u] = ldg16(y + (size_t)v * 8);
        ud[u] = ldg16(dout + (size_t)v * 8);
        if (MODE == 2) uo[u] = ldg16(out + (size_t)v * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const unsigned v = v0 + u * stride;
      if (v >= nvec) break;
      const int c0 = (int)(v % cv) * 8;
      const size_t off = (size_t)v * 8;
      float fy[8], fd[8], r[8];
      unpack8(uy[u], fy);
      unpack8(ud[u], fd);
      if (MODE == 2) {
        float fo[8];
        unpack8(uo[u], fo);
#pragma unroll
        for (int i = 0; i < 8; ++i) fd[i] = fo[i] > 0.f ? fd[i] : 0.f;
      }
      if (MODE == 1) {
        float sc[8], sh[8];
        ld8f(scale + c0, sc);
        ld8f(shift + c0, sh);
#pragma unroll
        for (int i = 0; i < 8; ++i) fd[i] = (fmaf(fy[i], sc[i], sh[i]) > 0.f) ? fd[i] : 0.f;
      }
      // MODE 3: `dout` already holds g (written by the reduction), no mask
      {
        float k[8];
        ld8f(coef + c0, k);
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = k[i] * fd[i];
        ld8f(coef + C + c0, k);
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] += k[i] * fy[i];
        ld8f(coef + 2 * C + c0, k);
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] += k[i];
      }
      if (acc_dy) {
        float prev[8];
        unpack8(*reinterpret_cast<const uint4*>(dy + off), prev);
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] += prev[i];
      }
      *reinterpret_cast<uint4*>(dy + off) = pack8(r);
      if (SKIP) {
        if (acc_dskip) {
          float prev[8];
          unpack8(*reinterpret_cast<const uint4*>(dskip + off), prev);
#pragma unroll
          for (int i = 0; i < 8; ++i) fd[i] += prev[i];
        }
        *reinterpret_cast<uint4*>(dskip + off) = pack8(fd);
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) relu_fwd_kernel(const __nv_bfloat16* __restrict__ x, long nvec,
                                                           __nv_bfloat16* __restrict__ y) {
  pdl_enter();
  for (long v = (long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.x * blockDim.x) {
    float f[8];
    unpack8(ldg16(x + v * 8), f);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = fmaxf(f[i], 0.f);
    *reinterpret_cast<uint4*>(y + v * 8) = pack8(f);
  }
}

__global__ void __launch_bounds__(kThreads) relu_bwd_kernel(const __nv_bfloat16* __restrict__ y,
                                                           const __nv_bfloat16* __restrict__ dy, long nvec,
                                                           __nv_bfloat16* __restrict__ dx, int acc) {
  pdl_enter();
  for (long v = (long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.x * blockDim.x) {
    float fy[8], fd[8];
    unpack8(ldg16(y + v * 8), fy);
    unpack8(ldg16(dy + v * 8), fd);
#pragma unroll
    for (int i = 0; i < 8; ++i) fd[i] = fy[i] > 0.f ? fd[i] : 0.f;
    if (acc) {
      float p[8];
      unpack8(*reinterpret_cast<const uint4*>(dx + v * 8), p);
#pragma unroll
      for (int i = 0; i < 8; ++i) fd[i] += p[i];
    }
    *reinterpret_cast<uint4*>(dx + v * 8) = pack8(fd);
  }
}

// ------------------------------------------------------------ pooling
// Compile-time k x k window (the stem's 3x3 / 2): all k*k 16-byte loads of an
// output vector are issued before any comparison (the loop form waits for
// each load in turn: 1.5 TB/s on the stem pool); out-of-image taps are
// masked, and the comparisons run in the same (r, s) order with the same
// strict '>' (first argmax), so outputs and indices are the loop form's bits.
template <int KW>
__global__ void __launch_bounds__(kThreads) maxpool_fwd_k_kernel(const __nv_bfloat16* __restrict__ x, PoolGeom g,
                                                                __nv_bfloat16* __restrict__ y,
                                                                uint8_t* __restrict__ idx) {
  pdl_enter();
  const int cv = g.C / 8;
  const unsigned total = (unsigned)g.N * g.P * g.Q * cv;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = (int)(i % (unsigned)cv);
    unsigned t = i / (unsigned)cv;
    const int q = (int)(t % (unsigned)g.Q);
    t /= (unsigned)g.Q;
    const int p = (int)(t % (unsigned)g.P);
    const int n = (int)(t / (unsigned)g.P);
    const int h0 = p * g.stride - g.pad, w0 = q * g.stride - g.pad;
    uint4 v[KW * KW];
    bool ok[KW * KW];
#pragma unroll
    for (int r = 0; r < KW; ++r)
#pragma unroll
      for (int s = 0; s < KW; ++s) {
        const int h = h0 + r, w = w0 + s;
        ok[r * KW + s] = h >= 0 && h < g.H && w >= 0 && w < g.W;
        v[r * KW + s] = ok[r * KW + s] ? ldg16(x + (((long)n * g.H + h) * g.W + w) * g.C + c8 * 8)
                                       : make_uint4(0u, 0u, 0u, 0u);
      }
    float m[8];
    uint32_t best[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m[k] = -INFINITY;
      best[k] = 0;
    }
#pragma unroll
    for (int j = 0; j < KW * KW; ++j) {
      if (!ok[j]) continue;
      float f[8];
      unpack8(v[j], f);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (f[k] > m[k]) {
          m[k] = f[k];
          best[k] = (uint32_t)j;
        }
    }
    *reinterpret_cast<uint4*>(y + (size_t)i * 8) = pack8(m);
    if (idx) {
      uint2 o;
      o.x = best[0] | (best[1] << 8) | (best[2] << 16) | (best[3] << 24);
      o.y = best[4] | (best[5] << 8) | (best[6] << 16) | (best[7] << 24);
      *reinterpret_cast<uint2*>(idx + (size_t)i * 8) = o;
    }
  }
}

// idx (optional): the first-argmax window position of every output, for the
// backward gather (same rule as maxpool_argmax_kernel)
__global__ void __launch_bounds__(kThreads) maxpool_fwd_kernel(const __nv_bfloat16* __restrict__ x, PoolGeom g,
                                                              __nv_bfloat16* __restrict__ y, uint8_t* __restrict__ idx) {
  pdl_enter();
  const int cv = g.C / 8;
  const unsigned total = (unsigned)g.N * g.P * g.Q * cv;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = (int)(i % (unsigned)cv);
    unsigned t = i / (unsigned)cv;
    const int q = (int)(t % (unsigned)g.Q);
    t /= (unsigned)g.Q;
    const int p = (int)(t % (unsigned)g.P);
    const int n = (int)(t / (unsigned)g.P);
    float m[8];
    uint32_t best[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m[k] = -INFINITY;
      best[k] = 0;
    }
    for (int r = 0; r < g.k; ++r) {
      const int h = p * g.stride - g.pad + r;
      if (h < 0 || h >= g.H) continue;
      for (int s = 0; s < g.k; ++s) {
        const int w = q * g.stride - g.pad + s;
        if (w < 0 || w >= g.W) continue;
        float f[8];
        unpack8(ldg16(x + (((long)n * g.H + h) * g.W + w) * g.C + c8 * 8), f);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (f[k] > m[k]) {
            m[k] = f[k];
            best[k] = (uint32_t)(r * g.k + s);
          }
      }
    }
    *reinterpret_cast<uint4*>(y + (size_t)i * 8) = pack8(m);
    if (idx) {
      uint2 o;
      o.x = best[0] | (best[1] << 8) | (best[2] << 16) | (best[3] << 24);
      o.y = best[4] | (best[5] << 8) | (best[6] << 16) | (best[7] << 24);
      *reinterpret_cast<uint2*>(idx + (size_t)i * 8) = o;
    }
  }
}

// Windowed average pooling (torch AvgPool2d, count_include_pad=True: the sum
// over the in-bounds taps is always divided by k*k).
__global__ void __launch_bounds__(kThreads) avgpool2d_fwd_kernel(const __nv_bfloat16* __restrict__ x, PoolGeom g,
                                                                __nv_bfloat16* __restrict__ y) {
  pdl_enter();
  const int cv = g.C / 8;
  const unsigned total = (unsigned)g.N * g.P * g.Q * cv;
  const float inv = 1.f / (float)(g.k * g.k);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = (int)(i % (unsigned)cv);
    unsigned t = i / (unsigned)cv;
    const int q = (int)(t % (unsigned)g.Q);
    t /= (unsigned)g.Q;
    const int p = (int)(t % (unsigned)g.P);
    const int n = (int)(t / (unsigned)g.P);
    float m[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = 0.f;
    for (int r = 0; r < g.k; ++r) {
      const int h = p * g.stride - g.pad + r;
      if (h < 0 || h >= g.H) continue;
      for (int s = 0; s < g.k; ++s) {
        const int w = q * g.stride - g.pad + s;
        if (w < 0 || w >= g.W) continue;
        float f[8];
        unpack8(ldg16(x + (((long)n * g.H + h) * g.W + w) * g.C + c8 * 8), f);
#pragma unroll
        for (int k = 0; k < 8; ++k) m[k] += f[k];
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] *= inv;
    *reinterpret_cast<uint4*>(y + (size_t)i * 8) = pack8(m);
  }
}

// Gather form of the backward (no atomics): every input pixel sums dy over
// the windows that cover it, in a fixed (p, q) order.
__global__ void __launch_bounds__(kThreads) avgpool2d_bwd_kernel(const __nv_bfloat16* __restrict__ dy, PoolGeom g,
                                                                __nv_bfloat16* __restrict__ dx, int acc) {
  pdl_enter();
  const int cv = g.C / 8;
  const unsigned total = (unsigned)g.N * g.H * g.W * cv;
  const float inv = 1.f / (float)(g.k * g.k);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = (int)(i % (unsigned)cv);
    unsigned t = i / (unsigned)cv;
    const int w = (int)(t % (unsigned)g.W);
    t /= (unsigned)g.W;
    const int h = (int)(t % (unsigned)g.H);
    const int n = (int)(t / (unsigned)g.H);
    // windows p with p*stride - pad <= h < p*stride - pad + k
    const int p0 = max(0, (h + g.pad - g.k + g.stride) / g.stride), p1 = min(g.P - 1, (h + g.pad) / g.stride);
    const int q0 = max(0, (w + g.pad - g.k + g.stride) / g.stride), q1 = min(g.Q - 1, (w + g.pad) / g.stride);
    float m[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] = 0.f;
    for (int p = p0; p <= p1; ++p)
      for (int q = q0; q <= q1; ++q) {
        float f[8];
        unpack8(ldg16(dy + (((long)n * g.P + p) * g.Q + q) * g.C + c8 * 8), f);
#pragma unroll
        for (int k = 0; k < 8; ++k) m[k] += f[k];
      }
#pragma unroll
    for (int k = 0; k < 8; ++k) m[k] *= inv;
    if (acc) {
      float prev[8];
      unpack8(*reinterpret_cast<const uint4*>(dx + (size_t)i * 8), prev);
#pragma unroll
      for (int k = 0; k < 8; ++k) m[k] += prev[k];
    }
    *reinterpret_cast<uint4*>(dx + (size_t)i * 8) = pack8(m);
  }
}

// Backward, pass 1: first argmax (row-major window position, ties to the
// first hit) of every window and channel, one byte each.
__global__ void __launch_bounds__(kThreads) maxpool_argmax_kernel(const __nv_bfloat16* __restrict__ x, PoolGeom g,
                                                                 uint8_t* __restrict__ idx) {
  pdl_enter();
  const int cv = g.C / 8;
  const unsigned total = (unsigned)g.N * g.P * g.Q * cv;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = (int)(i % (unsigned)cv);
    unsigned t = i / (unsigned)cv;
    const int q = (int)(t % (unsigned)g.Q);
    t /= (unsigned)g.Q;
    const int p = (int)(t % (unsigned)g.P);
    const int n = (int)(t / (unsigned)g.P);
    float m[8];
    uint32_t best[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      m[k] = -INFINITY;
      best[k] = 0;
    }
    for (int r = 0; r < g.k; ++r) {
      const int h = p * g.stride - g.pad + r;
      if (h < 0 || h >= g.H) continue;
      for (int s = 0; s < g.k; ++s) {
        const int w = q * g.stride - g.pad + s;
        if (w < 0 || w >= g.W) continue;
        float f[8];
        unpack8(ldg16(x + (((long)n * g.H + h) * g.W + w) * g.C + c8 * 8), f);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (f[k] > m[k]) {
            m[k] = f[k];
            best[k] = (uint32_t)(r * g.k + s);
          }
      }
    }
    uint2 o;
    o.x = best[0] | (best[1] << 8) | (best[2] << 16) | (best[3] << 24);
    o.y = best[4] | (best[5] << 8) | (best[6] << 16) | (best[7] << 24);
    *reinterpret_cast<uint2*>(idx + (size_t)i * 8) = o;
  }
}

// Backward, pass 2 (gather, no atomics): each input element sums, in fixed
// window order, dy of every covering window whose argmax it is.
__global__ void __launch_bounds__(kThreads) maxpool_bwd_kernel(const uint8_t* __restrict__ idx,
                                                              const __nv_bfloat16* __restrict__ dy, PoolGeom g,
                                                              __nv_bfloat16* __restrict__ dx, int acc) {
  pdl_enter();
  const int cv = g.C / 8;
  const unsigned total = (unsigned)g.N * g.H * g.W * cv;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = (int)(i % (unsigned)cv);
    unsigned t = i / (unsigned)cv;
    const int w = (int)(t % (unsigned)g.W);
    t /= (unsigned)g.W;
    const int h = (int)(t % (unsigned)g.H);
    const int n = (int)(t / (unsigned)g.H);
    float sum[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sum[k] = 0.f;
    // windows p with p*stride - pad <= h <= p*stride - pad + k - 1
    const int p_lo = max(0, (h + g.pad - g.k + g.stride) / g.stride);
    const int p_hi = min(g.P - 1, (h + g.pad) / g.stride);
    const int q_lo = max(0, (w + g.pad - g.k + g.stride) / g.stride);
    const int q_hi = min(g.Q - 1, (w + g.pad) / g.stride);
    for (int p = p_lo; p <= p_hi; ++p)
      for (int q = q_lo; q <= q_hi; ++q) {
        const long o = ((((long)n * g.P + p) * g.Q + q) * cv + c8);
        const uint2 iv = __ldg(reinterpret_cast<const uint2*>(idx + o * 8));
        const uint32_t self = (uint32_t)((h - (p * g.stride - g.pad)) * g.k + (w - (q * g.stride - g.pad)));
        float dv[8];
        unpack8(ldg16(dy + o * 8), dv);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t b = ((k < 4 ? iv.x : iv.y) >> (8 * (k & 3))) & 0xffu;
          if (b == self) sum[k] += dv[k];
        }
      }
    if (acc) {
      float pv[8];
      unpack8(*reinterpret_cast<const uint4*>(dx + (size_t)i * 8), pv);
#pragma unroll
      for (int k = 0; k < 8; ++k) sum[k] += pv[k];
    }
    *reinterpret_cast<uint4*>(dx + (size_t)i * 8) = pack8(sum);
  }
}

// Gather with a compile-time k x k / stride window: the (at most
// ceil(k / stride))^2 covering windows' index and dy loads are all issued
// before the sums, which run in the loop form's (p, q) order (same bits).
template <int KW, int KS, int CV>
__global__ void __launch_bounds__(kThreads) maxpool_bwd_k_kernel(const uint8_t* __restrict__ idx,
                                                                const __nv_bfloat16* __restrict__ dy, PoolGeom g,
                                                                __nv_bfloat16* __restrict__ dx, int acc) {
  pdl_enter();
  constexpr int NW = (KW + KS - 1) / KS;  // covering windows per dimension
  const int cv = CV > 0 ? CV : g.C / 8;   // compile-time vectors per pixel (the stem: 64 channels)
  const unsigned total = (unsigned)g.N * g.H * g.W * cv;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = (int)(i % (unsigned)cv);
    unsigned t = i / (unsigned)cv;
    const int w = (int)(t % (unsigned)g.W);
    t /= (unsigned)g.W;
    const int h = (int)(t % (unsigned)g.H);
    const int n = (int)(t / (unsigned)g.H);
    const int p_lo = max(0, (h + g.pad - KW + KS) / KS);
    const int p_hi = min(g.P - 1, (h + g.pad) / KS);
    const int q_lo = max(0, (w + g.pad - KW + KS) / KS);
    const int q_hi = min(g.Q - 1, (w + g.pad) / KS);
    uint2 iv[NW * NW];
    uint4 dv[NW * NW];
    bool ok[NW * NW];
#pragma unroll
    for (int a = 0; a < NW; ++a)
#pragma unroll
      for (int b = 0; b < NW; ++b) {
        const int p = p_lo + a, q = q_lo + b;
        const int j = a * NW + b;
        ok[j] = p <= p_hi && q <= q_hi;
        const long o = ((((long)n * g.P + p) * g.Q + q) * cv + c8);
        iv[j] = ok[j] ? __ldg(reinterpret_cast<const uint2*>(idx + o * 8)) : make_uint2(0xffffffffu, 0xffffffffu);
        dv[j] = ok[j] ? ldg16(dy + o * 8) : make_uint4(0u, 0u, 0u, 0u);
      }
    uint4 prev = make_uint4(0u, 0u, 0u, 0u);
    if (acc) prev = *reinterpret_cast<const uint4*>(dx + (size_t)i * 8);
    float sum[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sum[k] = 0.f;
#pragma unroll
    for (int j = 0; j < NW * NW; ++j) {
      if (!ok[j]) continue;
      const int p = p_lo + j / NW, q = q_lo + j % NW;
      const uint32_t self = (uint32_t)((h - (p * KS - g.pad)) * KW + (w - (q * KS - g.pad)));
      // all eight channels' argmax bytes against this pixel's window position
      // at once (0xff per matching byte); windows selecting none are skipped
      const uint32_t m0 = __vcmpeq4(iv[j].x, self * 0x01010101u), m1 = __vcmpeq4(iv[j].y, self * 0x01010101u);
      if ((m0 | m1) == 0u) continue;
      float d[8];
      unpack8(dv[j], d);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (((k < 4 ? m0 : m1) >> (8 * (k & 3))) & 1u) sum[k] += d[k];
    }
    if (acc) {
      float pv[8];
      unpack8(prev, pv);
#pragma unroll
      for (int k = 0; k < 8; ++k) sum[k] += pv[k];
    }
    *reinterpret_cast<uint4*>(dx + (size_t)i * 8) = pack8(sum);
  }
}

// Fused backward (argmax + gather in one pass, no index workspace): a block
// owns a T x T tile of windows of one image and the input pixels whose rows /
// columns fall in that tile's stride partition.  The input patch under the
// tile's windows (plus the hp low-side halo windows that also cover owned
// pixels) is staged in shared memory with batched 16-byte loads; phase 1
// finds each staged window's first argmax there and stages its dy; phase 2
// gives every owned input pixel the sum, in fixed (p, q) order, of dy over
// the covering windows whose argmax it is -- the same order, so the same
// bits, as the two-kernel form.
template <int KW, int KS>
__global__ void __launch_bounds__(kThreads) maxpool_bwd_tiled_kernel(const __nv_bfloat16* __restrict__ x,
                                                                    const __nv_bfloat16* __restrict__ dy, PoolGeom g,
                                                                    int T, __nv_bfloat16* __restrict__ dx, int acc) {
  pdl_enter();
  extern __shared__ __align__(16) uint8_t pool_s[];
  if (KW) g.k = KW;  // compile-time window / stride: divisions become shifts
  if (KS) g.stride = KS;
  const int cv = g.C / 8;
  const int hp = (g.k - 1) / g.stride;
  const int tiles_q = (g.Q + T - 1) / T, tiles_p = (g.P + T - 1) / T;
  const int WT = T + hp;                       // staged windows per side
  const int XT = (WT - 1) * g.stride + g.k;    // staged input pixels per side
  const int nwin = WT * WT;
  uint4* x_s = reinterpret_cast<uint4*>(pool_s);                                      // [XT][XT][cv]
  uint4* dy_s = x_s + (size_t)XT * XT * cv;                                           // [nwin][cv]
  uint2* ix_s = reinterpret_cast<uint2*>(dy_s + (size_t)nwin * cv);                   // [nwin][cv]
  for (int tile = blockIdx.x; tile < g.N * tiles_p * tiles_q; tile += gridDim.x) {
    const int tq = tile % tiles_q, tp = (tile / tiles_q) % tiles_p, n = tile / (tiles_q * tiles_p);
    const int p0 = tp * T, q0 = tq * T;
    const int hb = (p0 - hp) * g.stride - g.pad, wb = (q0 - hp) * g.stride - g.pad;  // patch origin
    __syncthreads();
    {
      // patch rows are contiguous runs of XT*cv vectors: per-thread column
      // index fixed, four rows' loads in flight
      const int rowv = XT * cv;
      for (int j = threadIdx.x; j < rowv; j += blockDim.x) {
        const int w = wb + j / cv;
        const bool okw = w >= 0 && w < g.W;
        const uint4* src = reinterpret_cast<const uint4*>(x) + ((long)n * g.H * g.W + wb) * cv + j;
        for (int r0 = 0; r0 < XT; r0 += 4) {
          uint4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int h = hb + r0 + u;
            v[u] = make_uint4(0u, 0u, 0u, 0u);
            if (r0 + u < XT && okw && h >= 0 && h < g.H) v[u] = __ldg(src + (long)h * g.W * cv);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (r0 + u < XT) x_s[(r0 + u) * rowv + j] = v[u];
        }
      }
      for (int i = threadIdx.x; i < nwin * cv; i += blockDim.x) {
        const int c8 = i % cv, wi = i / cv;
        const int p = p0 - hp + wi / WT, q = q0 - hp + wi % WT;
        if (p >= 0 && p < g.P && q >= 0 && q < g.Q) dy_s[i] = ldg16(dy + ((((long)n * g.P + p) * g.Q + q) * cv + c8) * 8);
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nwin * cv; i += blockDim.x) {
      const int c8 = i % cv, wi = i / cv;
      const int pr = wi / WT, qr = wi % WT;
      const int p = p0 - hp + pr, q = q0 - hp + qr;
      if (p < 0 || p >= g.P || q < 0 || q >= g.Q) continue;
      // first argmax, bf16x2 SIMD: strict '>' keeps the first hit (and
      // ignores NaN) like the scalar form; window positions as byte lanes
      uint32_t m[4] = {0xff80ff80u, 0xff80ff80u, 0xff80ff80u, 0xff80ff80u};  // -inf pairs
      uint32_t bx = 0, by = 0;
      for (int r = 0; r < g.k; ++r) {
        const int h = p * g.stride - g.pad + r;
        if (h < 0 || h >= g.H) continue;
        for (int s = 0; s < g.k; ++s) {
          const int w = q * g.stride - g.pad + s;
          if (w < 0 || w >= g.W) continue;
          const uint4 v = x_s[((pr * g.stride + r) * XT + qr * g.stride + s) * cv + c8];
          const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
          uint32_t gm[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            __nv_bfloat162 a2, b2;
            memcpy(&a2, &vv[t], 4);
            memcpy(&b2, &m[t], 4);
            gm[t] = __hgt2_mask(a2, b2);
            m[t] = (vv[t] & gm[t]) | (m[t] & ~gm[t]);
          }
          const uint32_t pos = (uint32_t)(r * g.k + s) * 0x01010101u;
          const uint32_t b0 = __byte_perm(gm[0], gm[1], 0x6420), b1 = __byte_perm(gm[2], gm[3], 0x6420);
          bx = (pos & b0) | (bx & ~b0);
          by = (pos & b1) | (by & ~b1);
        }
      }
      ix_s[i] = make_uint2(bx, by);
    }
    __syncthreads();
    // owned input rows / columns: the stride partition of this tile (the
    // first tile from 0, the last to the end)
    const int h_lo = tp == 0 ? 0 : p0 * g.stride - g.pad;
    const int h_hi = tp == tiles_p - 1 ? g.H : min(g.H, (p0 + T) * g.stride - g.pad);
    const int w_lo = tq == 0 ? 0 : q0 * g.stride - g.pad;
    const int w_hi = tq == tiles_q - 1 ? g.W : min(g.W, (q0 + T) * g.stride - g.pad);
    const int ow = max(0, w_hi - w_lo);
    const int row_items = ow * cv;
    // (c8, w) of a thread fixed per tile when the block covers whole rows
    const bool rows_fit = row_items > 0 && (int)blockDim.x % row_items == 0;
    const int owned = max(0, h_hi - h_lo) * row_items;
    const int c8f = rows_fit ? (int)threadIdx.x % cv : 0, wf = rows_fit ? w_lo + ((int)threadIdx.x / cv) % ow : 0;
    const int hstep = rows_fit ? (int)blockDim.x / row_items : 0;
    for (int j = threadIdx.x, it = 0; j < owned; j += blockDim.x, ++it) {
      int c8, w, h;
      if (rows_fit) {
        c8 = c8f, w = wf, h = h_lo + (int)threadIdx.x / row_items + it * hstep;  // j = threadIdx.x + it * blockDim.x
      } else {
        c8 = j % cv;
        const int t = j / cv;
        w = w_lo + t % ow, h = h_lo + t / ow;
      }
      float sum[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) sum[k] = 0.f;
      const int p_lo = max(0, (h + g.pad - g.k + g.stride) / g.stride);
      const int p_hi = min(g.P - 1, (h + g.pad) / g.stride);
      const int q_lo = max(0, (w + g.pad - g.k + g.stride) / g.stride);
      const int q_hi = min(g.Q - 1, (w + g.pad) / g.stride);
      for (int p = p_lo; p <= p_hi; ++p)
        for (int q = q_lo; q <= q_hi; ++q) {
          const int wi = (p - p0 + hp) * WT + (q - q0 + hp);
          const uint2 iv = ix_s[wi * cv + c8];
          const uint32_t self = (uint32_t)((h - (p * g.stride - g.pad)) * g.k + (w - (q * g.stride - g.pad)));
          // per-channel byte compare -> bf16 lane masks; adding a masked +0
          // leaves the fp32 sum bit-identical (it is never -0)
          const uint32_t mx = __vcmpeq4(iv.x, self * 0x01010101u), my = __vcmpeq4(iv.y, self * 0x01010101u);
          uint4 d = dy_s[wi * cv + c8];
          d.x &= __byte_perm(mx, 0, 0x1100);
          d.y &= __byte_perm(mx, 0, 0x3322);
          d.z &= __byte_perm(my, 0, 0x1100);
          d.w &= __byte_perm(my, 0, 0x3322);
          float dv[8];
          unpack8(d, dv);
#pragma unroll
          for (int k = 0; k < 8; ++k) sum[k] += dv[k];
        }
      __nv_bfloat16* o = dx + (((long)n * g.H + h) * g.W + w) * g.C + c8 * 8;
      if (acc) {
        float pv[8];
        unpack8(*reinterpret_cast<const uint4*>(o), pv);
#pragma unroll
        for (int k = 0; k < 8; ++k) sum[k] += pv[k];
      }
      *reinterpret_cast<uint4*>(o) = pack8(sum);
    }
  }
}

// global average pool: block per (n, 256-channel chunk); fixed-order sums
__global__ void __launch_bounds__(kThreads) avgpool_fwd_kernel(const __nv_bfloat16* __restrict__ x, int HW, int C,
                                                              __nv_bfloat16* __restrict__ out) {
  pdl_enter();
  const int n = blockIdx.x;
  const int c = blockIdx.y * kThreads + threadIdx.x;
  if (c >= C) return;
  float s = 0.f;
  const __nv_bfloat16* p = x + (long)n * HW * C + c;
  for (int i = 0; i < HW; ++i) s += __bfloat162float(p[(long)i * C]);
  out[(long)n * C + c] = __float2bfloat16_rn(s / (float)HW);
}

__global__ void __launch_bounds__(kThreads) avgpool_bwd_kernel(const __nv_bfloat16* __restrict__ dout, int HW, int C,
                                                              long nvec, __nv_bfloat16* __restrict__ dx, int acc) {
  pdl_enter();
  const float inv = 1.f / (float)HW;
  for (long v = (long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.x * blockDim.x) {
    const long e = v * 8;
    const int c0 = (int)(e % C);
    const long n = e / ((long)HW * C);
    float f[8];
    unpack8(ldg16(dout + n * C + c0), f);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] *= inv;
    if (acc) {
      float p[8];
      unpack8(*reinterpret_cast<const uint4*>(dx + e), p);
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] += p[i];
    }
    *reinterpret_cast<uint4*>(dx + e) = pack8(f);
  }
}

// ------------------------------------------------------------ loss
// One block per row: logsumexp in fp32; lse[n] saved for the backward.
__global__ void __launch_bounds__(kThreads) softmax_ce_fwd_kernel(const float* __restrict__ logits,
                                                                 const int* __restrict__ labels, int K,
                                                                 float* __restrict__ row_loss,
                                                                 float* __restrict__ lse_out) {
  pdl_enter();
  __shared__ float red[kThreads];
  const int n = blockIdx.x;
  const float* z = logits + (long)n * K;
  float m = -INFINITY;
  for (int k = threadIdx.x; k < K; k += kThreads) m = fmaxf(m, z[k]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  m = red[0];
  __syncthreads();
  float e = 0.f;
  for (int k = threadIdx.x; k < K; k += kThreads) e += expf(z[k] - m);
  red[threadIdx.x] = e;
  __syncthreads();
  for (int s = kThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const float lse = m + logf(red[0]);
    lse_out[n] = lse;
    row_loss[n] = lse - z[labels[n]];
  }
}

__global__ void mean_kernel(const float* __restrict__ v, int n, float* __restrict__ out) {
  pdl_enter();
  __shared__ float red[kThreads];
  float s = 0.f;
  for (int i = threadIdx.x; i < n; i += kThreads) s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = kThreads / 2; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0] / (float)n;
}

// dlogits = (softmax - onehot) / N ; fp32 and a bf16 copy [N, ldb]
__global__ void __launch_bounds__(kThreads) softmax_ce_bwd_kernel(const float* __restrict__ logits,
                                                                 const int* __restrict__ labels,
                                                                 const float* __restrict__ lse, int Nrows, int K,
                                                                 float* __restrict__ dlogits) {
  pdl_enter();
  const long total = (long)Nrows * K;
  const float invn = 1.f / (float)Nrows;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int n = (int)(i / K), k = (int)(i % K);
    float p = expf(logits[i] - lse[n]);
    if (k == labels[n]) p -= 1.f;
    dlogits[i] = p * invn;
  }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ x, long n, __nv_bfloat16* __restrict__ y) {
  pdl_enter();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    y[i] = __float2bfloat16_rn(x[i]);
}

__global__ void __launch_bounds__(kThreads) cast_f32_bf16_vec_kernel(const float* __restrict__ x, long nvec,
                                                                    __nv_bfloat16* __restrict__ y) {
  pdl_enter();
  for (long v = (long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.x * blockDim.x) {
    float f[8];
    ld8f(x + v * 8, f);
    *reinterpret_cast<uint4*>(y + v * 8) = pack8(f);
  }
}

// fp32 [R, C] -> bf16 [R, ldo] (pad columns untouched)
__global__ void cast_f32_bf16_2d_kernel(const float* __restrict__ x, int R, int C, int ldo,
                                        __nv_bfloat16* __restrict__ y) {
  pdl_enter();
  const long total = (long)R * C;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x)
    y[(i / C) * ldo + (i % C)] = __float2bfloat16_rn(x[i]);
}

// column sums of a bf16 [R, C] matrix, fixed order
__global__ void colsum_bf16_kernel(const __nv_bfloat16* __restrict__ x, int R, int C, float* __restrict__ out,
                                   int acc) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s = 0.f;
  for (int r = 0; r < R; ++r) s += __bfloat162float(x[(long)r * C + c]);
  out[c] = acc ? out[c] + s : s;
}

// column sums of an fp32 [R, C] matrix (bias gradient), fixed order
__global__ void colsum_f32_kernel(const float* __restrict__ x, int R, int C, float* __restrict__ out, int acc) {
  pdl_enter();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s = 0.f;
  for (int r = 0; r < R; ++r) s += x[(long)r * C + c];
  out[c] = acc ? out[c] + s : s;
}

// sum of split-K partials [splits][n] -> out (fixed order)
// float4 per thread, split loop unrolled by 4 so several loads are in flight;
// summation order z = 0, 1, ... is fixed (deterministic)
// Many splits over a small output (the weight gradients of the deep, narrow
// layers): 8 thread groups per output vector each sum every 8th split, then
// a fixed pairwise tree in shared memory combines them -- 8x the loads in
// flight, still one fixed summation order.
__global__ void __launch_bounds__(kThreads) reduce_splits_grouped_kernel(const float* __restrict__ parts, int splits,
                                                                        unsigned n4, float* __restrict__ out, int acc) {
  pdl_enter();
  __shared__ float4 sh[8][32];
  const float4* p4 = reinterpret_cast<const float4*>(parts);
  const unsigned lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const unsigned i = blockIdx.x * 32 + lane;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < n4)
    for (int z = (int)grp; z < splits; z += 8) {
      const float4 a = __ldg(p4 + (size_t)z * n4 + i);
      s.x += a.x;
      s.y += a.y;
      s.z += a.z;
      s.w += a.w;
    }
  sh[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && i < n4) {
    float4 r[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) r[g] = sh[g][lane];
#pragma unroll
    for (int w = 4; w > 0; w >>= 1)
#pragma unroll
      for (int g = 0; g < w; ++g) {
        r[g].x += r[g + w].x;
        r[g].y += r[g + w].y;
        r[g].z += r[g + w].z;
        r[g].w += r[g + w].w;
      }
    float4* o = reinterpret_cast<float4*>(out) + i;
    if (acc) {
      const float4 prev = *o;
      r[0].x += prev.x;
      r[0].y += prev.y;
      r[0].z += prev.z;
      r[0].w += prev.w;
    }
    *o = r[0];
  }
}

// Split-K finish for a bf16 activation output (conv fprop / dgrad of the
// deep, low-parallelism layers): out[m][c] (+)= bf16(sum_z parts[z][m][c]) in
// split order, and optionally the BN column sum / sum of squares of the
// stored bf16 values, one row per block (the conv's statistics slot layout).
// Block = (N/4 float4 lanes) x row groups over a contiguous row slab.
__global__ void __launch_bounds__(kThreads) reduce_splits_bf16_kernel(const float* __restrict__ parts, int splits,
                                                                     int M, int N, int rows_per_block,
                                                                     __nv_bfloat16* out, long ldc, int acc,
                                                                     float* __restrict__ stats) {
  pdl_enter();
  __shared__ float4 shs[kThreads], shq[kThreads];
  const int lanes = N / 4, groups = kThreads / lanes;
  const int t = threadIdx.x, lane = t % lanes, grp = t / lanes;
  const long MN4 = (long)M * lanes;
  const float4* p4 = reinterpret_cast<const float4*>(parts);
  float4 cs = make_float4(0.f, 0.f, 0.f, 0.f), cq = cs;
  const int r0 = blockIdx.x * rows_per_block, r1 = min(M, r0 + rows_per_block);
  if (grp < groups) {
    for (int r = r0 + grp; r < r1; r += groups) {
      const long i = (long)r * lanes + lane;
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int z = 0; z < splits; ++z) {
        const float4 a = __ldg(p4 + (long)z * MN4 + i);
        s.x += a.x;
        s.y += a.y;
        s.z += a.z;
        s.w += a.w;
      }
      __nv_bfloat16* o = out + (long)r * ldc + lane * 4;
      if (acc) {
        const uint2 pv = *reinterpret_cast<const uint2*>(o);
        const float2 p0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv.x));
        const float2 p1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pv.y));
        s.x += p0.x;
        s.y += p0.y;
        s.z += p1.x;
        s.w += p1.y;
      }
      const __nv_bfloat162 b0 = __floats2bfloat162_rn(s.x, s.y), b1 = __floats2bfloat162_rn(s.z, s.w);
      uint2 ov;
      ov.x = *reinterpret_cast<const uint32_t*>(&b0);
      ov.y = *reinterpret_cast<const uint32_t*>(&b1);
      *reinterpret_cast<uint2*>(o) = ov;
      if (stats) {
        const float2 f0 = __bfloat1622float2(b0), f1 = __bfloat1622float2(b1);
        cs.x += f0.x;
        cs.y += f0.y;
        cs.z += f1.x;
        cs.w += f1.y;
        cq.x = fmaf(f0.x, f0.x, cq.x);
        cq.y = fmaf(f0.y, f0.y, cq.y);
        cq.z = fmaf(f1.x, f1.x, cq.z);
        cq.w = fmaf(f1.y, f1.y, cq.w);
      }
    }
  }
  if (!stats) return;
  shs[t] = cs;
  shq[t] = cq;
  __syncthreads();
  if (grp == 0) {
    for (int g = 1; g < groups; ++g) {
      const float4 a = shs[g * lanes + lane], b = shq[g * lanes + lane];
      cs.x += a.x;
      cs.y += a.y;
      cs.z += a.z;
      cs.w += a.w;
      cq.x += b.x;
      cq.y += b.y;
      cq.z += b.z;
      cq.w += b.w;
    }
    float* row = stats + (long)blockIdx.x * 2 * N + lane * 4;
    row[0] = cs.x;
    row[1] = cs.y;
    row[2] = cs.z;
    row[3] = cs.w;
    row[N + 0] = cq.x;
    row[N + 1] = cq.y;
    row[N + 2] = cq.z;
    row[N + 3] = cq.w;
  }
}

__global__ void __launch_bounds__(kThreads) reduce_splits_kernel(const float* __restrict__ parts, int splits, long n4,
                                                                float* __restrict__ out, int acc) {
  pdl_enter();
  const float4* p4 = reinterpret_cast<const float4*>(parts);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    int z = 0;
    for (; z + 4 <= splits; z += 4) {
      const float4 a = __ldg(p4 + (long)z * n4 + i), b = __ldg(p4 + (long)(z + 1) * n4 + i);
      const float4 c = __ldg(p4 + (long)(z + 2) * n4 + i), d = __ldg(p4 + (long)(z + 3) * n4 + i);
      s.x = (((s.x + a.x) + b.x) + c.x) + d.x;
      s.y = (((s.y + a.y) + b.y) + c.y) + d.y;
      s.z = (((s.z + a.z) + b.z) + c.z) + d.z;
      s.w = (((s.w + a.w) + b.w) + c.w) + d.w;
    }
    for (; z < splits; ++z) {
      const float4 a = __ldg(p4 + (long)z * n4 + i);
      s.x += a.x;
      s.y += a.y;
      s.z += a.z;
      s.w += a.w;
    }
    float4* o = reinterpret_cast<float4*>(out) + i;
    if (acc) {
      const float4 prev = *o;
      s.x += prev.x;
      s.y += prev.y;
      s.z += prev.z;
      s.w += prev.w;
    }
    *o = s;
  }
}

// ------------------------------------------------------------ optimizer + layouts
// SGD with momentum and weight decay, 4 parameters per thread-iteration; when
// wb is given it also refreshes the bf16 GEMM copy of the weights in the same
// pass (n % 4 == 0, 16-byte aligned buffers).
__global__ void __launch_bounds__(kThreads) sgd_kernel(float* __restrict__ w, const float* __restrict__ g,
                                                      float* __restrict__ m, long n4,
                                                      const float* __restrict__ hyper,
                                                      __nv_bfloat16* __restrict__ wb) {
  pdl_enter();
  // lr, momentum, weight decay from device memory: a captured step graph
  // stays valid under a learning-rate schedule
  const float lr = __ldg(hyper), momentum = __ldg(hyper + 1), wd = __ldg(hyper + 2);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 wv = reinterpret_cast<float4*>(w)[i];
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    float4 mv = reinterpret_cast<float4*>(m)[i];
    float* wp = &wv.x;
    const float* gp = &gv.x;
    float* mp = &mv.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float d = gp[k] + wd * wp[k];
      const float v = momentum * mp[k] + d;
      mp[k] = v;
      wp[k] = wp[k] - lr * v;
    }
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(w)[i] = wv;
    if (wb) {
      uint2 o;
      o.x = pack_bf16_pair(wv.x, wv.y);
      o.y = pack_bf16_pair(wv.z, wv.w);
      reinterpret_cast<uint2*>(wb)[i] = o;
    }
  }
}

// fp32 [Cout][R][S][Cpad] -> bf16 same layout, and bf16 flipped transpose
// Wt[ci][R-1-r][S-1-s][co] with co padded to CoutPad.
__global__ void conv_weight_prep_kernel(const float* __restrict__ w, int Cout, int R, int S, int Cpad, int Cin,
                                        int CoutPad, __nv_bfloat16* __restrict__ wb, __nv_bfloat16* __restrict__ wt) {
  pdl_enter();
  const long total = (long)Cout * R * S * Cpad;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cpad);
    long t = i / Cpad;
    const int s = (int)(t % S);
    t /= S;
    const int r = (int)(t % R);
    const int co = (int)(t / R);
    const __nv_bfloat16 v = __float2bfloat16_rn(w[i]);
    wb[i] = v;
    if (wt && c < Cin) wt[(((long)c * R + (R - 1 - r)) * S + (S - 1 - s)) * CoutPad + co] = v;
  }
}

__global__ void __launch_bounds__(kThreads) weight_prep_batched_kernel(const WeightPrepLayer* __restrict__ tab,
                                                                      int layers, long total) {
  pdl_enter();
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    int lo = 0, hi = layers - 1;  // last layer with start <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tab[mid].start <= i) lo = mid;
      else hi = mid - 1;
    }
    const WeightPrepLayer& L = tab[lo];
    long e = i - L.start;
    if (e < L.n_copy) {  // coalesced copy in GEMM layout
      L.wb[e] = __float2bfloat16_rn(L.w[e]);
      continue;
    }
    e -= L.n_copy;  // transpose, iterated in output order: wt[ci][r'][s'][co]
    const int co = (int)(e % L.coutpad);
    long t = e / L.coutpad;
    const int s2 = (int)(t % L.S);
    t /= L.S;
    const int r2 = (int)(t % L.R);
    const int ci = (int)(t / L.R);
    float v = 0.f;
    if (co < L.cout) v = L.w[(((long)co * L.R + (L.R - 1 - r2)) * L.S + (L.S - 1 - s2)) * L.cpad + ci];
    L.wt[e] = __float2bfloat16_rn(v);
  }
}

// NCHW fp32 -> NHWC bf16 with zero channel padding to Cpad
__global__ void pack_input_kernel(const float* __restrict__ x, int N, int C, int H, int W, int Cpad,
                                  __nv_bfloat16* __restrict__ out) {
  pdl_enter();
  const long total = (long)N * H * W * Cpad;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int c = (int)(i % Cpad);
    long t = i / Cpad;
    const int w = (int)(t % W);
    t /= W;
    const int h = (int)(t % H);
    const int n = (int)(t / H);
    const float v = c < C ? x[(((long)n * C + c) * H + h) * W + w] : 0.f;
    out[i] = __float2bfloat16_rn(v);
  }
}

// one thread per pixel and group of 8 channels: plane reads are coalesced
// across the warp (consecutive w), the NHWC write is one 16-byte store
__global__ void pack_input_vec_kernel(const float* __restrict__ x, int N, int C, int H, int W, int Cpad,
                                      __nv_bfloat16* __restrict__ out) {
  pdl_enter();
  const long HW = (long)H * W;
  const int groups = Cpad / 8;
  const long total = (long)N * HW * groups;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const long pix = i % ((long)N * HW);
    const int grp = (int)(i / ((long)N * HW));
    const long n = pix / HW, hw = pix % HW;
    uint32_t w2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c0 = grp * 8 + 2 * j;
      const float a = c0 < C ? __ldg(x + (n * C + c0) * HW + hw) : 0.f;
      const float b = c0 + 1 < C ? __ldg(x + (n * C + c0 + 1) * HW + hw) : 0.f;
      w2[j] = pack_bf16_pair(a, b);
    }
    *reinterpret_cast<uint4*>(out + pix * Cpad + grp * 8) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
  }
}

// The common case (C <= 8 real channels -> one 16-byte group, H*W % 4 == 0):
// each thread packs four consecutive pixels of one image from one float4 per
// channel, 32-bit indexing.
__global__ void __launch_bounds__(kThreads) pack_input_q4_kernel(const float* __restrict__ x, int N, int C,
                                                                unsigned HW4, __nv_bfloat16* __restrict__ out) {
  pdl_enter();
  const unsigned total = (unsigned)N * HW4;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned n = i / HW4, q = i - n * HW4;
    float v[8][4];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < C) f = __ldg(reinterpret_cast<const float4*>(x + ((size_t)n * C + c) * HW4 * 4) + q);
      v[c][0] = f.x, v[c][1] = f.y, v[c][2] = f.z, v[c][3] = f.w;
    }
    uint4* o = reinterpret_cast<uint4*>(out) + (size_t)i * 4;
#pragma unroll
    for (int p = 0; p < 4; ++p)
      o[p] = make_uint4(pack_bf16_pair(v[0][p], v[1][p]), pack_bf16_pair(v[2][p], v[3][p]),
                        pack_bf16_pair(v[4][p], v[5][p]), pack_bf16_pair(v[6][p], v[7][p]));
  }
}

// explicit im2col for thin-channel convs: out[m][k], k = (r*S + s)*C + c, K
// padded with zeros to Kpad.
// One thread per (output pixel, 8 consecutive k): a single 16-byte store;
// the pixel decode is done once per thread.
__global__ void __launch_bounds__(kThreads) im2col_kernel(const __nv_bfloat16* __restrict__ x, ConvShape g, int Kpad,
                                                         __nv_bfloat16* __restrict__ out) {
  pdl_enter();
  const int kv = Kpad / 8;
  const long total = (long)g.N * g.P * g.Q * kv;
  const int Kreal = g.R * g.S * g.C;
  const unsigned short* xs = reinterpret_cast<const unsigned short*>(x);
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int k0 = (int)(i % kv) * 8;
    const long m = i / kv;
    const int q = (int)(m % g.Q);
    const long t = m / g.Q;
    const int p = (int)(t % g.P);
    const int n = (int)(t / g.P);
    const int h0 = p * g.stride - g.pad, w0 = q * g.stride - g.pad;
    const unsigned short* base = xs + (long)n * g.H * g.W * g.Cs;
    unsigned short e[8];
    int c = k0 % g.C, rs = k0 / g.C;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      unsigned short v = 0;
      if (k0 + j < Kreal) {
        const int s = rs % g.S, r = rs / g.S;
        const int h = h0 + r, w = w0 + s;
        if (h >= 0 && h < g.H && w >= 0 && w < g.W) v = __ldg(base + ((long)h * g.W + w) * g.Cs + c);
      }
      e[j] = v;
      if (++c == g.C) {
        c = 0;
        ++rs;
      }
    }
    uint4 o;
    o.x = e[0] | ((uint32_t)e[1] << 16);
    o.y = e[2] | ((uint32_t)e[3] << 16);
    o.z = e[4] | ((uint32_t)e[5] << 16);
    o.w = e[6] | ((uint32_t)e[7] << 16);
    *reinterpret_cast<uint4*>(out + m * Kpad + k0) = o;
  }
}

// Window-staged im2col (the stem's few-channel conv): a block takes a run of
// `rpb` consecutive output rows p0.. of one image and stages the
// (rpb-1)*stride + R input rows they read in shared memory, zero-padded to
// W + 2*pad columns and COMPACT -- only the C real channels per pixel, so the
// (r, s, c) K order of a tap row is contiguous and consecutive K groups of a
// warp read consecutive shared-memory words (no bank conflicts; the padded
// 16-byte pixels made 4-way conflicts).  The global loads of a window are
// issued four per thread before any store.  Then the rpb Q x Kpad slabs are
// written with coalesced 16-byte stores.
__global__ void __launch_bounds__(kThreads) im2col_rows_kernel(const __nv_bfloat16* __restrict__ x, ConvShape g,
                                                              int Kpad, int rpb, __nv_bfloat16* __restrict__ out) {
  pdl_enter();
  extern __shared__ __align__(16) unsigned short rows_s[];  // [window rows][W + 2 pad][C], then the k table
  const int Wp = g.W + 2 * g.pad;
  const int cv = g.Cs / 8;  // 16-byte vectors per stored pixel
  const int kv = Kpad / 8;
  const int Kreal = g.R * g.S * g.C;
  const int win = (rpb - 1) * g.stride + g.R;
  // k -> offset of (r, s, c) in the staged rows relative to the output
  // pixel's first column of its first window row (-1: K padding)
  int* ktab = reinterpret_cast<int*>(rows_s + (((long)win * Wp * g.C + 7) & ~7L));
  for (int k = threadIdx.x; k < Kpad; k += blockDim.x) {
    const int c = k % g.C, rs = k / g.C, s = rs % g.S, r = rs / g.S;
    ktab[k] = k < Kreal ? (r * Wp + s) * g.C + c : -1;
  }
  const int runs_per_img = (g.P + rpb - 1) / rpb;
  const int step = blockDim.x / kv;
  const int kg = threadIdx.x % kv;
  for (int run = blockIdx.x; run < g.N * runs_per_img; run += gridDim.x) {
    const int n = run / runs_per_img, p0 = (run % runs_per_img) * rpb;
    const int np = min(rpb, g.P - p0);
    const int h0 = p0 * g.stride - g.pad;
    const int rows = (np - 1) * g.stride + g.R;
    const int rowv = Wp * cv;  // 16-byte vectors per staged row
    const uint4* xv = reinterpret_cast<const uint4*>(x) + (long)n * g.H * g.W * cv;
    __syncthreads();  // the previous run's slabs are written
    // four rows' loads in flight per thread, then the compact stores
    for (int j = threadIdx.x; j < rowv; j += blockDim.x) {
      const int c8 = cv == 1 ? 0 : j % cv, wp = cv == 1 ? j : j / cv, w = wp - g.pad;
      const bool win_w = w >= 0 && w < g.W;
      for (int r0 = 0; r0 < rows; r0 += 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int h = h0 + r0 + u;
          v[u] = make_uint4(0u, 0u, 0u, 0u);
          if (r0 + u < rows && win_w && h >= 0 && h < g.H) v[u] = __ldg(xv + ((long)h * g.W + w) * cv + c8);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (r0 + u >= rows) break;
          const uint32_t wv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
          unsigned short* dst = rows_s + ((long)(r0 + u) * Wp + wp) * g.C + c8 * 8;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c8 * 8 + c < g.C) dst[c] = (unsigned short)(wv[c >> 1] >> ((c & 1) * 16));
        }
      }
    }
    __syncthreads();
    // each thread owns one 8-wide K group (its 8 gather offsets stay in
    // registers) and walks the output pixels; consecutive threads write
    // consecutive 16-byte vectors of a pixel's K row
    if ((int)threadIdx.x < step * kv) {
      // K padding: offset 0 and a zero mask instead of a per-element select
      int off[8];
      uint32_t mask[4];
#pragma unroll
      for (int j = 0; j < 8; ++j) off[j] = max(ktab[kg * 8 + j], 0);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        mask[j] = (ktab[kg * 8 + 2 * j] >= 0 ? 0xffffu : 0u) | (ktab[kg * 8 + 2 * j + 1] >= 0 ? 0xffff0000u : 0u);
      const bool all_pad = (mask[0] | mask[1] | mask[2] | mask[3]) == 0u;
      for (int pp = 0; pp < np; ++pp) {
        const unsigned short* base = rows_s + pp * g.stride * Wp * g.C;
        uint4* o = reinterpret_cast<uint4*>(out + ((long)n * g.P + p0 + pp) * g.Q * Kpad);
        for (int q = threadIdx.x / kv; q < g.Q; q += step) {
          uint4 val = make_uint4(0u, 0u, 0u, 0u);
          if (!all_pad) {
            const unsigned short* px = base + q * g.stride * g.C;
            uint32_t e[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) e[j] = px[off[j]];
            val = make_uint4(__byte_perm(e[0], e[1], 0x5410) & mask[0], __byte_perm(e[2], e[3], 0x5410) & mask[1],
                             __byte_perm(e[4], e[5], 0x5410) & mask[2], __byte_perm(e[6], e[7], 0x5410) & mask[3]);
          }
          o[q * kv + kg] = val;
        }
      }
    }
  }
}

// zero-inserted (stride-dilated) copy of dy: U[n][p*s][q*s] = dy[n][p][q]
__global__ void __launch_bounds__(kThreads) zero_insert_kernel(const __nv_bfloat16* __restrict__ dy, int N, int P,
                                                              int Q, int C, int Hu, int Wu, int stride,
                                                              __nv_bfloat16* __restrict__ u) {
  pdl_enter();
  const int cv = C / 8;
  const long total = (long)N * Hu * Wu * cv;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int c8 = (int)(i % cv);
    long t = i / cv;
    const int w = (int)(t % Wu);
    t /= Wu;
    const int h = (int)(t % Hu);
    const int n = (int)(t / Hu);
    uint4 v = make_uint4(0, 0, 0, 0);
    if (h % stride == 0 && w % stride == 0 && h / stride < P && w / stride < Q)
      v = ldg16(dy + (((long)n * P + h / stride) * Q + w / stride) * C + c8 * 8);
    *reinterpret_cast<uint4*>(u + i * 8) = v;
  }
}

// channel concat c = [a | b] and its backward
// (index type I: 32-bit unsigned whenever the vector count allows -- a 64-bit
// division per 16-byte vector made these copies instruction-bound)
template <typename I>
__global__ void __launch_bounds__(kThreads) concat_kernel(const __nv_bfloat16* __restrict__ a, int Ca,
                                                         const __nv_bfloat16* __restrict__ b, int Cb, long M,
                                                         __nv_bfloat16* __restrict__ c) {
  pdl_enter();
  const int Cc = Ca + Cb, cv = Cc / 8;
  const I total = (I)(M * cv);
  for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const size_t m = (size_t)(i / (I)cv);
    const int ch = (int)(i % (I)cv) * 8;
    if (ch < Ca) {
      if (a) *reinterpret_cast<uint4*>(c + m * Cc + ch) = ldg16(a + m * Ca + ch);
    } else if (b) {
      *reinterpret_cast<uint4*>(c + m * Cc + ch) = ldg16(b + m * Cb + (ch - Ca));
    }
  }
}

template <typename I>
__global__ void __launch_bounds__(kThreads) split_grad_kernel(const __nv_bfloat16* __restrict__ dc, int Ca, int Cb,
                                                             long M, __nv_bfloat16* __restrict__ da, int acc_a,
                                                             __nv_bfloat16* __restrict__ db, int acc_b) {
  pdl_enter();
  const int Cc = Ca + Cb, cv = Cc / 8;
  const I total = (I)(M * cv);
  for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
    const size_t m = (size_t)(i / (I)cv);
    const int ch = (int)(i % (I)cv) * 8;
    float f[8];
    unpack8(ldg16(dc + m * Cc + ch), f);
    __nv_bfloat16* dst;
    int acc;
    if (ch < Ca) {
      dst = da ? da + m * Ca + ch : nullptr;
      acc = acc_a;
    } else {
      dst = db ? db + m * Cb + (ch - Ca) : nullptr;
      acc = acc_b;
    }
    if (!dst) continue;
    if (acc) {
      float p[8];
      unpack8(*reinterpret_cast<const uint4*>(dst), p);
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] += p[k];
    }
    *reinterpret_cast<uint4*>(dst) = pack8(f);
  }
}

__global__ void __launch_bounds__(kThreads) add_bf16_kernel(const __nv_bfloat16* __restrict__ a, long nvec,
                                                           __nv_bfloat16* __restrict__ dst) {
  pdl_enter();
  for (long v = (long)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (long)gridDim.x * blockDim.x) {
    float x[8], y[8];
    unpack8(ldg16(a + v * 8), x);
    unpack8(*reinterpret_cast<const uint4*>(dst + v * 8), y);
#pragma unroll
    for (int i = 0; i < 8; ++i) y[i] += x[i];
    *reinterpret_cast<uint4*>(dst + v * 8) = pack8(y);
  }
}

long rows_per_block_for(long M, int blocks) { return (M + blocks - 1) / blocks; }

// Channel chunk of a column reduction's blocks (blockIdx.y): all of C when
// C <= 2048, else 2048; halved (while it divides C, down to 256 channels)
// until the grid holds two waves -- the deep 14x14 / 7x7 BNs have few rows,
// so rows alone gave them 25-98 blocks on 148 SMs.  0 = no valid chunking.
int reduce_chunk(int C, int blocks) {
  int cw = C <= 2048 ? C : 2048;
  if (C % cw) return 0;
  while ((long)blocks * (C / cw) < 2 * 148 && cw >= 512 && (cw / 2) % 8 == 0 && C % (cw / 2) == 0) cw /= 2;
  return cw;
}

// Timing experiments only (results become wrong): RFK_ABLATE bit mask skips
// kernels to bound what removing them could save -- 1 forward BN finalize,
// 2 backward BN finalize, 4 backward BN reduce, 8 forward BN apply,
// 16 backward BN apply.
// RFK_G_EARLY=0: the residual-add BN backward re-derives g in the apply pass
bool g_early_off() {
  static const bool off = [] {
    const char* e = std::getenv("RFK_G_EARLY");
    return e && std::atoi(e) == 0;
  }();
  return off;
}

int ablate() {
  static const int m = [] {
    const char* e = std::getenv("RFK_ABLATE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

}  // namespace

// ============================================================ launchers
int colstats_blocks(long M) {
  // one full wave (3 resident blocks per SM), each with >= 64 rows
  long b = (M + 63) / 64;
  if (b > 148 * 3) b = 148 * 3;
  return (int)(b < 1 ? 1 : b);
}

cudaError_t colstats(const __nv_bfloat16* x, long M, int C, float* partials, int blocks, cudaStream_t st) {
  const int cw = reduce_chunk(C, blocks);
  if (C % 8 || cw == 0) return cudaErrorInvalidValue;
  dim3 grid(blocks, C / cw);
  RFK_CHECK_LAUNCH(launch_k(colstats_kernel<0>, grid, kThreads, 0, st, x, M, C, rows_per_block_for(M, blocks), partials,
                            cw));
  return cudaGetLastError();
}

cudaError_t bn_finalize(const float* partials, int parts, int C, long count, const float* gamma, const float* beta,
                        float eps, float* mean, float* invstd, float* scale, float* shift, float* run_mean,
                        float* run_var, float momentum, bool update_running, cudaStream_t st) {
  if (ablate() & 1) return cudaSuccess;
  RFK_CHECK_LAUNCH(launch_k(bn_finalize_kernel, (C + 31) / 32, dim3(32, kFinY), 0, st, partials, parts, C, (float)count, gamma, beta, eps, mean,
                                                            invstd, scale, shift, run_mean, run_var, momentum,
                                                            update_running ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t bn_finalize_gather(const BnGatherBlock* table, int C, long count, const float* gamma, const float* beta,
                               float eps, float* mean, float* invstd, float* scale, float* shift, float* run_mean,
                               float* run_var, float momentum, cudaStream_t st) {
  if (C % 32) return cudaErrorInvalidValue;
  RFK_CHECK_LAUNCH(launch_k(bn_finalize_gather_kernel, C / 32, dim3(32, kFinY), 0, st, table, C, (float)count, gamma,
                            beta, eps, mean, invstd, scale, shift, run_mean, run_var, momentum));
  return cudaGetLastError();
}

cudaError_t bn_apply(const __nv_bfloat16* y, const __nv_bfloat16* skip, const float* scale, const float* shift,
                     bool relu, long M, int C, __nv_bfloat16* out, cudaStream_t st) {
  const long nvec = M * C / 8;
  if (nvec >= (1L << 31)) return cudaErrorInvalidValue;
  if (ablate() & 8) return cudaSuccess;
  const int g = grid_for(nvec, kThreads * kVec, 148 * 8);
  const unsigned nv = (unsigned)nvec;
  if (skip) {
    if (relu) RFK_CHECK_LAUNCH(launch_k(bn_apply_kernel<true, true>, g, kThreads, 0, st, y, skip, scale, shift, nv, C, out));
    else RFK_CHECK_LAUNCH(launch_k(bn_apply_kernel<true, false>, g, kThreads, 0, st, y, skip, scale, shift, nv, C, out));
  } else {
    if (relu) RFK_CHECK_LAUNCH(launch_k(bn_apply_kernel<false, true>, g, kThreads, 0, st, y, skip, scale, shift, nv, C, out));
    else RFK_CHECK_LAUNCH(launch_k(bn_apply_kernel<false, false>, g, kThreads, 0, st, y, skip, scale, shift, nv, C, out));
  }
  return cudaGetLastError();
}

cudaError_t bn_backward_from_rows(const __nv_bfloat16* y, const __nv_bfloat16* dout, const float* gamma,
                                  const float* mean, const float* invstd, const float* scale, const float* shift,
                                  long M, int C, const float* rows, int parts, float* coef, float* dgamma,
                                  float* dbeta, __nv_bfloat16* dy, bool acc_dy, cudaStream_t st) {
  const long nvec = M * C / 8;
  if (C % 8 || nvec >= (1L << 31)) return cudaErrorInvalidValue;
  if (!(ablate() & 2))
    RFK_CHECK_LAUNCH(launch_k(bn_bwd_finalize_kernel, (C + 31) / 32, dim3(32, kFinY), 0, st, rows, parts, C,
                              (float)M, gamma, mean, invstd, dgamma, dbeta, coef));
  if (ablate() & 16) return cudaGetLastError();
  const int g = grid_for(nvec, kThreads * 2, 148 * 4);
  RFK_CHECK_LAUNCH(launch_k(bn_bwd_apply_kernel<1, false>, g, kThreads, 0, st, y, dout,
                            static_cast<const __nv_bfloat16*>(nullptr), scale, shift, coef, (unsigned)nvec, C, dy,
                            acc_dy ? 1 : 0, static_cast<__nv_bfloat16*>(nullptr), 0));
  return cudaGetLastError();
}

cudaError_t bn_backward(const __nv_bfloat16* y, const __nv_bfloat16* dout, const __nv_bfloat16* out, int mask_mode,
                        const float* gamma, const float* mean, const float* invstd, const float* scale,
                        const float* shift, long M, int C, float* partials, int blocks, float* coef, float* dgamma,
                        float* dbeta, __nv_bfloat16* dy, bool acc_dy, __nv_bfloat16* dskip, bool acc_dskip,
                        cudaStream_t st) {
  const int cw = reduce_chunk(C, blocks);
  if (C % 8 || cw == 0 || mask_mode < 0 || mask_mode > 2) return cudaErrorInvalidValue;
  const long nvec = M * C / 8;
  if (nvec >= (1L << 31)) return cudaErrorInvalidValue;
  dim3 grid(blocks, C / cw);
  const long rpb = rows_per_block_for(M, blocks);
  // residual add whose skip gradient is written (not accumulated): the
  // reduction stores g there, and the apply reads g back (7 passes over the
  // tensor instead of 8: dout and out are read once, not twice)
  const bool g_early = mask_mode == 2 && dskip && !acc_dskip && !g_early_off();
  __nv_bfloat16* gout = g_early ? dskip : nullptr;
  if (!(ablate() & 4)) switch (mask_mode) {
    case 0: RFK_CHECK_LAUNCH(launch_k(bn_bwd_reduce_kernel<0>, grid, kThreads, 0, st, y, dout, out, mean, scale, shift, M, C, rpb, partials, gout, cw)); break;
    case 1: RFK_CHECK_LAUNCH(launch_k(bn_bwd_reduce_kernel<1>, grid, kThreads, 0, st, y, dout, out, mean, scale, shift, M, C, rpb, partials, gout, cw)); break;
    default: RFK_CHECK_LAUNCH(launch_k(bn_bwd_reduce_kernel<2>, grid, kThreads, 0, st, y, dout, out, mean, scale, shift, M, C, rpb, partials, gout, cw));
  }
  if (!(ablate() & 2)) RFK_CHECK_LAUNCH(launch_k(bn_bwd_finalize_kernel, (C + 31) / 32, dim3(32, kFinY), 0, st, partials, blocks, C, (float)M, gamma, mean, invstd,
                                                                dgamma, dbeta, coef));
  const int g = grid_for(nvec, kThreads * 2, 148 * 4);  // one wave at 4 blocks per SM
  const unsigned nv = (unsigned)nvec;
  const int ad = acc_dy ? 1 : 0, as = acc_dskip ? 1 : 0;
#define RF_BWD_APPLY(MODE, SKIP) \
  RFK_CHECK_LAUNCH(launch_k(bn_bwd_apply_kernel<MODE, SKIP>, g, kThreads, 0, st, y, dout, out, scale, shift, coef, nv, C, dy, ad, dskip, as))
  if (ablate() & 16) {
  } else if (g_early) {
    const __nv_bfloat16* gbuf = dskip;
    RFK_CHECK_LAUNCH(launch_k(bn_bwd_apply_kernel<3, false>, g, kThreads, 0, st, y, gbuf, out, scale, shift, coef, nv,
                              C, dy, ad, static_cast<__nv_bfloat16*>(nullptr), 0));
  } else if (dskip) {
    switch (mask_mode) {
      case 0: RF_BWD_APPLY(0, true); break;
      case 1: RF_BWD_APPLY(1, true); break;
      default: RF_BWD_APPLY(2, true);
    }
  } else {
    switch (mask_mode) {
      case 0: RF_BWD_APPLY(0, false); break;
      case 1: RF_BWD_APPLY(1, false); break;
      default: RF_BWD_APPLY(2, false);
    }
  }
#undef RF_BWD_APPLY
  return cudaGetLastError();
}

cudaError_t relu_fwd(const __nv_bfloat16* x, long n, __nv_bfloat16* y, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(relu_fwd_kernel, grid_for(n / 8, kThreads * 4), kThreads, 0, st, x, n / 8, y));
  return cudaGetLastError();
}

cudaError_t relu_bwd(const __nv_bfloat16* y, const __nv_bfloat16* dy, long n, __nv_bfloat16* dx, bool acc,
                     cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(relu_bwd_kernel, grid_for(n / 8, kThreads * 4), kThreads, 0, st, y, dy, n / 8, dx, acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t maxpool_fwd(const __nv_bfloat16* x, const PoolGeom& g, __nv_bfloat16* y, cudaStream_t st, uint8_t* idx) {
  if ((long)g.N * g.H * g.W * (g.C / 8) >= (1L << 31)) return cudaErrorInvalidValue;  // 32-bit indexing
  if (idx && g.k * g.k > 256) return cudaErrorInvalidValue;
  const long work = (long)g.N * g.P * g.Q * (g.C / 8);
  if (g.k == 3)
    RFK_CHECK_LAUNCH(launch_k(maxpool_fwd_k_kernel<3>, grid_for(work, kThreads * 2), kThreads, 0, st, x, g, y, idx));
  else if (g.k == 2)
    RFK_CHECK_LAUNCH(launch_k(maxpool_fwd_k_kernel<2>, grid_for(work, kThreads * 2), kThreads, 0, st, x, g, y, idx));
  else
    RFK_CHECK_LAUNCH(launch_k(maxpool_fwd_kernel, grid_for(work, kThreads * 2), kThreads, 0, st, x, g, y, idx));
  return cudaGetLastError();
}

cudaError_t maxpool_bwd_from_idx(const uint8_t* idx, const __nv_bfloat16* dy, const PoolGeom& g, __nv_bfloat16* dx,
                                 bool acc, cudaStream_t st) {
  if ((long)g.N * g.H * g.W * (g.C / 8) >= (1L << 31)) return cudaErrorInvalidValue;  // 32-bit indexing
  const long work = (long)g.N * g.H * g.W * (g.C / 8);
  if (g.k == 3 && g.stride == 2 && g.C == 64)
    RFK_CHECK_LAUNCH(launch_k(maxpool_bwd_k_kernel<3, 2, 8>, grid_for(work, kThreads * 2), kThreads, 0, st, idx, dy, g, dx,
                              acc ? 1 : 0));
  else if (g.k == 3 && g.stride == 2)
    RFK_CHECK_LAUNCH(launch_k(maxpool_bwd_k_kernel<3, 2, 0>, grid_for(work, kThreads * 2), kThreads, 0, st, idx, dy, g, dx,
                              acc ? 1 : 0));
  else if (g.k == 2 && g.stride == 2)
    RFK_CHECK_LAUNCH(launch_k(maxpool_bwd_k_kernel<2, 2, 0>, grid_for(work, kThreads * 2), kThreads, 0, st, idx, dy, g, dx,
                              acc ? 1 : 0));
  else if (g.k == 3 && g.stride == 1)
    RFK_CHECK_LAUNCH(launch_k(maxpool_bwd_k_kernel<3, 1, 0>, grid_for(work, kThreads * 2), kThreads, 0, st, idx, dy, g, dx,
                              acc ? 1 : 0));
  else
    RFK_CHECK_LAUNCH(launch_k(maxpool_bwd_kernel, grid_for(work, kThreads * 2), kThreads, 0, st, idx, dy, g, dx,
                              acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t avgpool2d_fwd(const __nv_bfloat16* x, const PoolGeom& g, __nv_bfloat16* y, cudaStream_t st) {
  if ((long)g.N * g.H * g.W * (g.C / 8) >= (1L << 31)) return cudaErrorInvalidValue;  // 32-bit indexing
  if (g.C % 8) return cudaErrorInvalidValue;
  const long work = (long)g.N * g.P * g.Q * (g.C / 8);
  RFK_CHECK_LAUNCH(launch_k(avgpool2d_fwd_kernel, grid_for(work, kThreads * 2), kThreads, 0, st, x, g, y));
  return cudaGetLastError();
}

cudaError_t avgpool2d_bwd(const __nv_bfloat16* dy, const PoolGeom& g, __nv_bfloat16* dx, bool acc, cudaStream_t st) {
  if ((long)g.N * g.H * g.W * (g.C / 8) >= (1L << 31)) return cudaErrorInvalidValue;  // 32-bit indexing
  if (g.C % 8) return cudaErrorInvalidValue;
  const long work = (long)g.N * g.H * g.W * (g.C / 8);
  RFK_CHECK_LAUNCH(launch_k(avgpool2d_bwd_kernel, grid_for(work, kThreads * 2), kThreads, 0, st, dy, g, dx, acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t maxpool_bwd(const __nv_bfloat16* x, const __nv_bfloat16* y, const __nv_bfloat16* dy, const PoolGeom& g,
                        __nv_bfloat16* dx, bool acc, void* idx_ws, cudaStream_t st) {
  if ((long)g.N * g.H * g.W * (g.C / 8) >= (1L << 31)) return cudaErrorInvalidValue;  // 32-bit indexing
  (void)y;
  if (g.k * g.k > 256) return cudaErrorInvalidValue;
  // fused single pass when the window tile (8x8, else smaller) fits in 48 KB
  const int cv = g.C / 8, hp = (g.k - 1) / g.stride;
  static const int t_max = std::getenv("RFK_POOL_TILE") ? std::atoi(std::getenv("RFK_POOL_TILE")) : 8;
  for (int T = t_max; T >= 2; T /= 2) {
    const long xt = (long)(T + hp - 1) * g.stride + g.k;
    const long smem = xt * xt * cv * 16 + (long)(T + hp) * (T + hp) * cv * 24;
    if (smem > 64 * 1024 || std::getenv("RFK_POOL_TWO_PASS")) continue;
    auto kern = g.k == 3 && g.stride == 2 ? maxpool_bwd_tiled_kernel<3, 2>
                : g.k == 2 && g.stride == 2 ? maxpool_bwd_tiled_kernel<2, 2> : maxpool_bwd_tiled_kernel<0, 0>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const long tiles = (long)g.N * ((g.P + T - 1) / T) * ((g.Q + T - 1) / T);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
    const long blocks = std::min<long>(tiles, 148L * std::max(1, per_sm));
    RFK_CHECK_LAUNCH(launch_k(kern, (int)blocks, kThreads, smem, st, x, dy, g, T, dx, acc ? 1 : 0));
    return cudaGetLastError();
  }
  uint8_t* idx = static_cast<uint8_t*>(idx_ws);
  const long wins = (long)g.N * g.P * g.Q * (g.C / 8);
  RFK_CHECK_LAUNCH(launch_k(maxpool_argmax_kernel, grid_for(wins, kThreads * 2), kThreads, 0, st, x, g, idx));
  const long work = (long)g.N * g.H * g.W * (g.C / 8);
  RFK_CHECK_LAUNCH(launch_k(maxpool_bwd_kernel, grid_for(work, kThreads * 2), kThreads, 0, st, idx, dy, g, dx, acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t avgpool_fwd(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* out, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(avgpool_fwd_kernel, dim3(N, (C + kThreads - 1) / kThreads), kThreads, 0, st, x, HW, C, out));
  return cudaGetLastError();
}

cudaError_t avgpool_bwd(const __nv_bfloat16* dout, int N, int HW, int C, __nv_bfloat16* dx, bool acc,
                        cudaStream_t st) {
  const long nvec = (long)N * HW * C / 8;
  RFK_CHECK_LAUNCH(launch_k(avgpool_bwd_kernel, grid_for(nvec, kThreads * 4), kThreads, 0, st, dout, HW, C, nvec, dx, acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t softmax_ce_fwd(const float* logits, const int* labels, int N, int K, float* row_loss, float* lse,
                           float* loss, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(softmax_ce_fwd_kernel, N, kThreads, 0, st, logits, labels, K, row_loss, lse));
  RFK_CHECK_LAUNCH(launch_k(mean_kernel, 1, kThreads, 0, st, row_loss, N, loss));
  return cudaGetLastError();
}

cudaError_t softmax_ce_bwd(const float* logits, const int* labels, const float* lse, int N, int K, float* dlogits,
                           cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(softmax_ce_bwd_kernel, grid_for((long)N * K, kThreads), kThreads, 0, st, logits, labels, lse, N, K, dlogits));
  return cudaGetLastError();
}

cudaError_t cast_f32_bf16(const float* x, long n, __nv_bfloat16* y, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(cast_f32_bf16_kernel, grid_for(n, kThreads * 4), kThreads, 0, st, x, n, y));
  return cudaGetLastError();
}

cudaError_t cast_f32_bf16_vec(const float* x, long n, __nv_bfloat16* y, cudaStream_t st) {
  if (n % 8) return cudaErrorInvalidValue;
  RFK_CHECK_LAUNCH(launch_k(cast_f32_bf16_vec_kernel, grid_for(n / 8, kThreads * 4), kThreads, 0, st, x, n / 8, y));
  return cudaGetLastError();
}

cudaError_t cast_f32_bf16_2d(const float* x, int R, int C, int ldo, __nv_bfloat16* y, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(cast_f32_bf16_2d_kernel, grid_for((long)R * C, kThreads * 4), kThreads, 0, st, x, R, C, ldo, y));
  return cudaGetLastError();
}

cudaError_t colsum_bf16(const __nv_bfloat16* x, int R, int C, float* out, bool acc, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(colsum_bf16_kernel, (C + kThreads - 1) / kThreads, kThreads, 0, st, x, R, C, out, acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t colsum_f32(const float* x, int R, int C, float* out, bool acc, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(colsum_f32_kernel, (C + kThreads - 1) / kThreads, kThreads, 0, st, x, R, C, out, acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t reduce_splits_bf16(const float* parts, int splits, int M, int N, __nv_bfloat16* out, long ldc, bool acc,
                               float* stats, int max_blocks, cudaStream_t st) {
  if (N % 4 || N / 4 > kThreads || ldc % 4) return cudaErrorInvalidValue;
  const int groups = kThreads / (N / 4);
  int blocks = (M + groups * 4 - 1) / (groups * 4);  // >= 4 rows per thread
  blocks = std::max(1, std::min(blocks, max_blocks));
  const int rpb = (M + blocks - 1) / blocks;
  blocks = (M + rpb - 1) / rpb;
  RFK_CHECK_LAUNCH(launch_k(reduce_splits_bf16_kernel, blocks, kThreads, 0, st, parts, splits, M, N, rpb, out, ldc,
                            acc ? 1 : 0, stats));
  return cudaGetLastError();
}

cudaError_t reduce_splits(const float* parts, int splits, long n, float* out, bool acc, cudaStream_t st) {
  if (n % 4) return cudaErrorInvalidValue;
  if (splits >= 8 && n / 4 < (1L << 31)) {
    RFK_CHECK_LAUNCH(launch_k(reduce_splits_grouped_kernel, (int)((n / 4 + 31) / 32), kThreads, 0, st, parts, splits,
                              (unsigned)(n / 4), out, acc ? 1 : 0));
    return cudaGetLastError();
  }
  RFK_CHECK_LAUNCH(launch_k(reduce_splits_kernel, grid_for(n / 4, kThreads, 148 * 8), kThreads, 0, st, parts, splits, n / 4, out,
                                                                               acc ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t sgd_update(float* w, const float* g, float* m, long n, const float* hyper, __nv_bfloat16* wb,
                       cudaStream_t st) {
  if (n % 4) return cudaErrorInvalidValue;
  RFK_CHECK_LAUNCH(launch_k(sgd_kernel, grid_for(n / 4, kThreads * 2), kThreads, 0, st, w, g, m, n / 4, hyper, wb));
  return cudaGetLastError();
}

cudaError_t conv_weight_prep(const float* w, int Cout, int R, int S, int Cpad, int Cin, int CoutPad,
                             __nv_bfloat16* wb, __nv_bfloat16* wt, cudaStream_t st) {
  const long total = (long)Cout * R * S * Cpad;
  RFK_CHECK_LAUNCH(launch_k(conv_weight_prep_kernel, grid_for(total, kThreads * 4), kThreads, 0, st, w, Cout, R, S, Cpad, Cin, CoutPad, wb,
                                                                              wt));
  return cudaGetLastError();
}

cudaError_t weight_prep_batched(const WeightPrepLayer* table_dev, int layers, long total, cudaStream_t st) {
  if (layers <= 0 || total <= 0) return cudaSuccess;
  RFK_CHECK_LAUNCH(launch_k(weight_prep_batched_kernel, grid_for(total, kThreads * 8, 148 * 16), kThreads, 0, st, table_dev, layers, total));
  return cudaGetLastError();
}

cudaError_t pack_input(const float* x, int N, int C, int H, int W, int Cpad, __nv_bfloat16* out, cudaStream_t st) {
  const long hw = (long)H * W;
  if (Cpad == 8 && C <= 8 && hw % 4 == 0 && (long)N * hw < (1L << 31) &&
      reinterpret_cast<uintptr_t>(x) % 16 == 0) {
    RFK_CHECK_LAUNCH(launch_k(pack_input_q4_kernel, grid_for((long)N * hw / 4, kThreads), kThreads, 0, st, x, N, C,
                              (unsigned)(hw / 4), out));
    return cudaGetLastError();
  }
  if (Cpad % 8 == 0) {
    const long work = (long)N * H * W * (Cpad / 8);
    RFK_CHECK_LAUNCH(launch_k(pack_input_vec_kernel, grid_for(work, kThreads * 2), kThreads, 0, st, x, N, C, H, W, Cpad, out));
    return cudaGetLastError();
  }
  const long total = (long)N * H * W * Cpad;
  RFK_CHECK_LAUNCH(launch_k(pack_input_kernel, grid_for(total, kThreads * 4), kThreads, 0, st, x, N, C, H, W, Cpad, out));
  return cudaGetLastError();
}

cudaError_t im2col(const __nv_bfloat16* x, const ConvShape& g, int Kpad, __nv_bfloat16* out, cudaStream_t st) {
  if (Kpad % 8) return cudaErrorInvalidValue;
  // rows per run: the largest <= 8 whose compact window fits 48 KB
  const long row_bytes = (long)(g.W + 2 * g.pad) * g.C * 2;
  auto smem_for = [&](int r) { return ((((long)(r - 1) * g.stride + g.R) * row_bytes + 15) & ~15L) + (long)Kpad * 4; };
  int rpb = 8;
  while (rpb > 1 && smem_for(rpb) > 48 * 1024) --rpb;
  const long win_smem = smem_for(rpb);
  if (g.Cs % 8 == 0 && win_smem <= 96 * 1024 && Kpad / 8 <= kThreads) {
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(im2col_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      attr_set = true;
    }
    const long runs = (long)g.N * ((g.P + rpb - 1) / rpb);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, im2col_rows_kernel, kThreads, win_smem);
    const long blocks = std::min<long>(runs, 148L * std::max(1, per_sm));
    RFK_CHECK_LAUNCH(launch_k(im2col_rows_kernel, (int)blocks, kThreads, win_smem, st, x, g, Kpad, rpb, out));
    return cudaGetLastError();
  }
  const long total = (long)g.N * g.P * g.Q * (Kpad / 8);
  RFK_CHECK_LAUNCH(launch_k(im2col_kernel, grid_for(total, kThreads * 2, 148 * 32), kThreads, 0, st, x, g, Kpad, out));
  return cudaGetLastError();
}

// Zero fill / copy of 16-byte-aligned device ranges as PDL kernels: inside
// the step's graph a memset or memcpy node is not a programmatic dependent of
// the kernel before it, so it would cut the launch / prologue overlap of the
// kernel chain around it (a 51 MB memset before a strided 1x1 dgrad, the
// residual add's skip copy).
__global__ void __launch_bounds__(kThreads) fill_zero_kernel(uint4* __restrict__ p, unsigned long n16) {
  pdl_enter();
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  for (unsigned long i = blockIdx.x * (unsigned long)blockDim.x + threadIdx.x; i < n16;
       i += (unsigned long)gridDim.x * blockDim.x)
    p[i] = z;
}

__global__ void __launch_bounds__(kThreads) copy16_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                          unsigned long n16) {
  pdl_enter();
  unsigned long i = blockIdx.x * (unsigned long)blockDim.x + threadIdx.x;
  const unsigned long step = (unsigned long)gridDim.x * blockDim.x;
  for (; i + 3 * step < n16; i += 4 * step) {  // four 16-byte loads in flight
    const uint4 a = __ldg(src + i), b = __ldg(src + i + step), c = __ldg(src + i + 2 * step),
                d = __ldg(src + i + 3 * step);
    dst[i] = a;
    dst[i + step] = b;
    dst[i + 2 * step] = c;
    dst[i + 3 * step] = d;
  }
  for (; i < n16; i += step) dst[i] = __ldg(src + i);
}

cudaError_t fill_zero(void* p, long bytes, cudaStream_t st) {
  if (bytes <= 0) return cudaSuccess;
  if ((reinterpret_cast<uintptr_t>(p) & 15) || (bytes & 15)) return cudaMemsetAsync(p, 0, bytes, st);
  const unsigned long n16 = (unsigned long)bytes / 16;
  RFK_CHECK_LAUNCH(launch_k(fill_zero_kernel, grid_for((long)n16, kThreads * 4, 148 * 8), kThreads, 0, st,
                            static_cast<uint4*>(p), n16));
  return cudaGetLastError();
}

cudaError_t copy_bytes(void* dst, const void* src, long bytes, cudaStream_t st) {
  if (bytes <= 0) return cudaSuccess;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) || (bytes & 15))
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st);
  const unsigned long n16 = (unsigned long)bytes / 16;
  RFK_CHECK_LAUNCH(launch_k(copy16_kernel, grid_for((long)n16, kThreads * 4, 148 * 8), kThreads, 0, st,
                            static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16));
  return cudaGetLastError();
}

cudaError_t zero_insert(const __nv_bfloat16* dy, int N, int P, int Q, int C, int Hu, int Wu, int stride,
                        __nv_bfloat16* u, cudaStream_t st) {
  const long work = (long)N * Hu * Wu * (C / 8);
  RFK_CHECK_LAUNCH(launch_k(zero_insert_kernel, grid_for(work, kThreads * 4), kThreads, 0, st, dy, N, P, Q, C, Hu, Wu, stride, u));
  return cudaGetLastError();
}

cudaError_t concat(const __nv_bfloat16* a, int Ca, const __nv_bfloat16* b, int Cb, long M, __nv_bfloat16* c,
                   cudaStream_t st) {
  const long work = M * ((Ca + Cb) / 8);
  if (work < (1L << 31))
    RFK_CHECK_LAUNCH(launch_k(concat_kernel<unsigned>, grid_for(work, kThreads * 4), kThreads, 0, st, a, Ca, b, Cb, M, c));
  else
    RFK_CHECK_LAUNCH(launch_k(concat_kernel<long>, grid_for(work, kThreads * 4), kThreads, 0, st, a, Ca, b, Cb, M, c));
  return cudaGetLastError();
}

cudaError_t split_grad(const __nv_bfloat16* dc, int Ca, int Cb, long M, __nv_bfloat16* da, bool acc_a,
                       __nv_bfloat16* db, bool acc_b, cudaStream_t st) {
  const long work = M * ((Ca + Cb) / 8);
  if (work < (1L << 31))
    RFK_CHECK_LAUNCH(launch_k(split_grad_kernel<unsigned>, grid_for(work, kThreads * 4), kThreads, 0, st, dc, Ca, Cb, M, da,
                              acc_a ? 1 : 0, db, acc_b ? 1 : 0));
  else
    RFK_CHECK_LAUNCH(launch_k(split_grad_kernel<long>, grid_for(work, kThreads * 4), kThreads, 0, st, dc, Ca, Cb, M, da,
                              acc_a ? 1 : 0, db, acc_b ? 1 : 0));
  return cudaGetLastError();
}

cudaError_t add_bf16(const __nv_bfloat16* a, long n, __nv_bfloat16* dst, cudaStream_t st) {
  RFK_CHECK_LAUNCH(launch_k(add_bf16_kernel, grid_for(n / 8, kThreads * 4), kThreads, 0, st, a, n / 8, dst));
  return cudaGetLastError();
}

}  // namespace rfk
