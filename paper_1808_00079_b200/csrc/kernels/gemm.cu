// Warp-specialised tcgen05 GEMM / implicit-GEMM convolution for sm_100a.
//
//   warp 0      TMA producer (one elected lane): A and B tiles -> smem ring
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: TMEM -> registers -> global, optional fused
//               per-column statistics (BatchNorm sum / sum of squares)
//
// Tiles: BLOCK_M = 128 output rows, BLOCK_N in {64, 128, 256}, BLOCK_K = 64
// (one 128-byte swizzle row of bf16).  Operands are staged with TMA in
// 128-byte-swizzled layouts, K-major or MN-major, and read by tcgen05.mma
// straight from shared memory; the fp32 accumulator lives in TMEM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>

#include "kernels/kernels.h"
#include "kernels/ptx.cuh"

namespace rfk {

namespace {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr int kThreads = 192;
constexpr int kTileA = kBlockM * kBlockK * 2;  // 16 KB

struct alignas(64) KParams {
  CUtensorMap ta;  // 64-byte aligned, must be first
  CUtensorMap tb;
  int M, N, K;
  int num_kb;          // total K blocks
  int kb_per_split;
  int a_kind, b_kind;
  // im2col geometry (for whichever operand is im2col)
  int g_P, g_Q, g_pad_h, g_pad_w, g_sh, g_sw, g_S, g_cblocks;
  // epilogue
  void* out;
  long ldc;
  int out_f32, accumulate_out;
  const float* bias;
  float* stats;
  long split_stride;
  int remap, rP, rQ, rH, rW, rsh, rsw;
  int stages;  // smem ring depth (<= Cfg::kStages); fewer for short K so more CTAs share an SM
};

template <int BN>
struct Cfg {
  static constexpr int kTileB = BN * kBlockK * 2;
  static constexpr int kStage = kTileA + kTileB;
  static constexpr int kStages = (BN == 64) ? 8 : (BN == 128 ? 6 : 4);
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kSmem = kStages * kStage + 1024 /*align slack*/ + 256 /*barriers*/;
};

// Decode a flattened output-pixel index into im2col TMA base coordinates.
__device__ __forceinline__ void pixel_base(const KParams& p, int m, int& w, int& h, int& n) {
  const int q = m % p.g_Q;
  const int t = m / p.g_Q;
  const int pp = t % p.g_P;
  n = t / p.g_P;
  w = q * p.g_sw - p.g_pad_w;
  h = pp * p.g_sh - p.g_pad_h;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ KParams p) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nst = p.stages;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + nst * C::kStage);
  uint64_t* empty = full + nst;
  uint64_t* tmem_full = empty + nst;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  float* red = reinterpret_cast<float*>(tmem_slot + 4);  // unused scratch

  const uint32_t warp = warp_id();
  const int m0 = blockIdx.x * kBlockM;
  const int n0 = blockIdx.y * BN;
  const int kb_begin = blockIdx.z * p.kb_per_split;
  const int kb_end = min(p.num_kb, kb_begin + p.kb_per_split);
  (void)red;

  if (warp == 0 && elect_one()) {
    tma_prefetch(&p.ta);
    tma_prefetch(&p.tb);
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      int aw = 0, ah = 0, an = 0;
      if (p.a_kind == (int)Operand::Im2colK) pixel_base(p, m0, aw, ah, an);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = kb_begin; kb < kb_end; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::kStage;
        uint8_t* sb = sa + kTileA;
        mbar_arrive_expect_tx(&full[stage], C::kStage);
        // A operand
        switch (p.a_kind) {
          case (int)Operand::KMajor2D:
            tma_load_2d(sa, &p.ta, &full[stage], kb * kBlockK, m0);
            break;
          case (int)Operand::MNMajor2D:
            tma_load_2d(sa, &p.ta, &full[stage], m0, kb * kBlockK);
            tma_load_2d(sa + kTileA / 2, &p.ta, &full[stage], m0 + 64, kb * kBlockK);
            break;
          default: {  // Im2colK: K block -> (tap, channel block)
            const int tap = kb / p.g_cblocks, cb = kb - tap * p.g_cblocks;
            const int r = tap / p.g_S, s = tap - r * p.g_S;
            tma_load_im2col(sa, &p.ta, &full[stage], cb * 64, aw, ah, an, (uint16_t)s, (uint16_t)r);
          }
        }
        // B operand
        switch (p.b_kind) {
          case (int)Operand::KMajor2D:
            tma_load_2d(sb, &p.tb, &full[stage], kb * kBlockK, n0);
            break;
          case (int)Operand::MNMajor2D:
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * 8192, &p.tb, &full[stage], n0 + 64 * j, kb * kBlockK);
            break;
          default: {  // Im2colMN: K block = 64 output pixels, MN = (tap, channel)
            int bw, bh, bn;
            pixel_base(p, kb * kBlockK, bw, bh, bn);
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) {
              const int nb = n0 / 64 + j;
              const int tap = nb / p.g_cblocks, cb = nb - tap * p.g_cblocks;
              const int r = tap / p.g_S, s = tap - r * p.g_S;
              tma_load_im2col(sb + j * 8192, &p.tb, &full[stage], cb * 64, bw, bh, bn, (uint16_t)s, (uint16_t)r);
            }
          }
        }
        if (++stage == nst) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const bool a_mn = p.a_kind == (int)Operand::MNMajor2D;
    const bool b_mn = p.b_kind == (int)Operand::MNMajor2D || p.b_kind == (int)Operand::Im2colMN;
    const uint32_t idesc = umma_idesc_bf16(kBlockM, BN, a_mn, b_mn);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb_begin; kb < kb_end; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(smem + stage * C::kStage);
        const uint32_t sb = sa + kTileA;
#pragma unroll
        for (int kk = 0; kk < kBlockK / 16; ++kk) {
          const uint64_t da = a_mn ? umma_desc_sw128(sa + kk * 2048, 8192, 1024)
                                   : umma_desc_sw128(sa + kk * 32, 16, 1024);
          const uint64_t db = b_mn ? umma_desc_sw128(sb + kk * 2048, 8192, 1024)
                                   : umma_desc_sw128(sb + kk * 32, 16, 1024);
          umma_bf16(tmem, da, db, idesc, (kb > kb_begin || kk > 0) ? 1u : 0u);
        }
        umma_commit(&empty[stage]);
        if (kb + 1 == kb_end) umma_commit(tmem_full);
      }
      __syncwarp();
      if (++stage == nst) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..5)
    const uint32_t quarter = warp & 3;
    const int row_local = quarter * 32 + lane_id();
    const int m = m0 + row_local;
    const bool row_ok = m < p.M;
    const bool empty_k = kb_end <= kb_begin;
    if (!empty_k) {
      mbar_wait(tmem_full, 0);
      tc_fence_after();
    }
    long out_row = m;
    if (p.remap && row_ok) {
      const int q = m % p.rQ, t = m / p.rQ, pp = t % p.rP, nn = t / p.rP;
      out_row = (long)nn * p.rH * p.rW + (long)(pp * p.rsh) * p.rW + (long)q * p.rsw;
    }
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      if (!empty_k) {
        tmem_ld32(tmem + ((quarter * 32u) << 16) + (uint32_t)c0, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) r[i] = 0u;
      }
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
      const int col0 = n0 + c0;
      if (p.bias) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += (col0 + i < p.N) ? p.bias[col0 + i] : 0.f;
      }
      if (row_ok) {
        if (p.out_f32) {
          float* dst = reinterpret_cast<float*>(p.out) + (long)blockIdx.z * p.split_stride + out_row * p.ldc + col0;
          if (col0 + 32 <= p.N) {
            if (p.accumulate_out) {
#pragma unroll
              for (int i = 0; i < 32; ++i) dst[i] += v[i];
            } else {
#pragma unroll
              for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            }
          } else {
            for (int i = 0; i < 32 && col0 + i < p.N; ++i) dst[i] = p.accumulate_out ? dst[i] + v[i] : v[i];
          }
        } else {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + (long)blockIdx.z * p.split_stride +
                               out_row * p.ldc + col0;
          if (p.accumulate_out) {
            if (col0 + 32 <= p.N) {
#pragma unroll
              for (int i = 0; i < 32; i += 8) {
                const uint4 o = *reinterpret_cast<const uint4*>(dst + i);
                const __nv_bfloat162* ob = reinterpret_cast<const __nv_bfloat162*>(&o);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float2 f = __bfloat1622float2(ob[j]);
                  v[i + 2 * j] += f.x;
                  v[i + 2 * j + 1] += f.y;
                }
              }
            } else {
              for (int i = 0; i < 32 && col0 + i < p.N; ++i) v[i] += __bfloat162float(dst[i]);
            }
          }
          if (col0 + 32 <= p.N) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 w;
              w.x = pack_bf16(v[i], v[i + 1]);
              w.y = pack_bf16(v[i + 2], v[i + 3]);
              w.z = pack_bf16(v[i + 4], v[i + 5]);
              w.w = pack_bf16(v[i + 6], v[i + 7]);
              *reinterpret_cast<uint4*>(dst + i) = w;
            }
          } else {
            for (int i = 0; i < 32 && col0 + i < p.N; ++i) dst[i] = __float2bfloat16_rn(v[i]);
          }
        }
      }
      if (p.stats) {
        // Column sums over this warp's 32 rows by a halving butterfly: after
        // 5 rounds lane l holds column l's total (31 shuffles per 32 columns).
        float s[32], q2[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          // statistics of the values actually stored (bf16-rounded), so the
          // BatchNorm that reads them back normalises exactly what it sees
          const float sv = p.out_f32 ? v[i] : __bfloat162float(__float2bfloat16_rn(v[i]));
          s[i] = row_ok ? sv : 0.f;
          q2[i] = s[i] * s[i];
        }
        const uint32_t lane = lane_id();
#pragma unroll
        for (int half = 16; half >= 1; half >>= 1) {
          const bool upper = (lane & half) != 0;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            // lanes with bit `half` set keep the upper half of the live window
            const float send_s = upper ? s[i] : s[i + half];
            const float send_q = upper ? q2[i] : q2[i + half];
            const float got_s = __shfl_xor_sync(0xffffffffu, send_s, half);
            const float got_q = __shfl_xor_sync(0xffffffffu, send_q, half);
            const float keep_s = upper ? s[i + half] : s[i];
            const float keep_q = upper ? q2[i + half] : q2[i];
            s[i] = keep_s + got_s;
            q2[i] = keep_q + got_q;
          }
        }
        // lane l now owns column c0 + l of this warp's 32 rows
        const int col = col0 + (int)lane;
        float* st = p.stats + (long)blockIdx.x * 2 * p.N;
        float* part = st;  // per-warp partials combined through shared memory below
        (void)part;
        __shared__ float red_s[4][32], red_q[4][32];
        red_s[quarter][lane] = s[0];
        red_q[quarter][lane] = q2[0];
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (quarter == 0 && col < p.N) {
          // fixed order over the four row quarters: deterministic
          const float ts = ((red_s[0][lane] + red_s[1][lane]) + red_s[2][lane]) + red_s[3][lane];
          const float tq = ((red_q[0][lane] + red_q[1][lane]) + red_q[2][lane]) + red_q[3][lane];
          st[col] = ts;
          st[p.N + col] = tq;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

// ------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_encode_im2col = nullptr;
std::once_flag g_once;
int g_driver_version = 0;

void load_driver_entry_points() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(fn);
    cudaDriverGetVersion(&g_driver_version);
  });
}

bool encode_2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
               uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode_tiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_im2col(CUtensorMap* m, const void* ptr, const ConvGeom& g, uint32_t pixels) {
  cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
  cuuint64_t strides[3] = {(cuuint64_t)g.C * 2, (cuuint64_t)g.W * g.C * 2, (cuuint64_t)g.H * g.W * g.C * 2};
  // bounding box of the receptive-field bases: [-pad, dim + pad - (filter-1))
  int lower[2] = {-g.pad_w, -g.pad_h};
  int upper[2] = {g.pad_w - (g.S - 1), g.pad_h - (g.R - 1)};
  cuuint32_t es[4] = {1, (cuuint32_t)g.stride_w, (cuuint32_t)g.stride_h, 1};
  CUresult r = g_encode_im2col(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, lower,
                               upper, 64, pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  // Small-tensor descriptor quirk on drivers <= 13.1 (same workaround as
  // CUTLASS copy_traits_sm90_im2col.hpp): clear bit 21 of word 1.
  const uint64_t bytes = (uint64_t)g.N * g.H * g.W * g.C * 2;
  if (g_driver_version <= 13010 && bytes < 131072) reinterpret_cast<uint64_t*>(m)[1] &= ~(1ull << 21);
  return true;
}

template <int BN>
cudaError_t launch_bn(KParams& kp, int m_tiles, int n_tiles, int splits, cudaStream_t st) {
  using C = Cfg<BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // ring depth: enough to cover this launch's K loop (a deeper ring only
  // costs residency), at least 2 so loads overlap MMAs
  kp.stages = std::max(2, std::min(C::kStages, kp.kb_per_split));
  const int smem = kp.stages * C::kStage + 1024 + 256;
  dim3 grid(m_tiles, n_tiles, splits);
  gemm_kernel<BN><<<grid, kThreads, smem, st>>>(kp);
  return cudaGetLastError();
}

}  // namespace

int gemm_m_tiles(const GemmDesc& d) { return (d.M + kBlockM - 1) / kBlockM; }

cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t stream) {
  load_driver_entry_points();
  if (!g_encode_tiled || !g_encode_im2col) return cudaErrorNotSupported;
  if (d.M <= 0 || d.N <= 0) return cudaSuccess;
  int bn = d.block_n;
  if (bn == 0) bn = d.N <= 64 ? 64 : (d.N <= 128 ? 128 : 256);
  if (d.b_kind == Operand::MNMajor2D || d.b_kind == Operand::Im2colMN) bn = bn < 64 ? 64 : bn;
  if (bn != 64 && bn != 128 && bn != 256) return cudaErrorInvalidValue;

  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.M = d.M;
  kp.N = d.N;
  kp.K = d.K;
  kp.a_kind = (int)d.a_kind;
  kp.b_kind = (int)d.b_kind;
  const ConvGeom* geo = nullptr;
  bool ok = true;
  switch (d.a_kind) {
    case Operand::KMajor2D:
      ok = encode_2d(&kp.ta, d.a, d.K, d.M, d.a_ld, 64, kBlockM);
      kp.num_kb = (d.K + 63) / 64;
      break;
    case Operand::MNMajor2D:
      ok = encode_2d(&kp.ta, d.a, d.M, d.K, d.a_ld, 64, 64);
      kp.num_kb = (d.K + 63) / 64;
      break;
    case Operand::Im2colK:
      geo = &d.a_geom;
      ok = encode_im2col(&kp.ta, d.a, d.a_geom, kBlockM);
      kp.num_kb = d.a_geom.R * d.a_geom.S * ((d.a_geom.C + 63) / 64);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  if (!ok) return cudaErrorInvalidValue;
  switch (d.b_kind) {
    case Operand::KMajor2D:
      ok = encode_2d(&kp.tb, d.b, (uint64_t)(d.a_kind == Operand::Im2colK ? (long)kp.num_kb * 64 : d.K), d.N, d.b_ld,
                     64, bn);
      break;
    case Operand::MNMajor2D:
      ok = encode_2d(&kp.tb, d.b, d.b_extent > 0 ? d.b_extent : d.N, d.K, d.b_ld, 64, 64);
      break;
    case Operand::Im2colMN:
      geo = &d.b_geom;
      ok = encode_im2col(&kp.tb, d.b, d.b_geom, 64);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  if (!ok) return cudaErrorInvalidValue;
  if (geo) {
    kp.g_P = geo->P;
    kp.g_Q = geo->Q;
    kp.g_pad_h = geo->pad_h;
    kp.g_pad_w = geo->pad_w;
    kp.g_sh = geo->stride_h;
    kp.g_sw = geo->stride_w;
    kp.g_S = geo->S;
    kp.g_cblocks = (geo->C + 63) / 64;
  }
  const int splits = d.splits < 1 ? 1 : d.splits;
  kp.kb_per_split = (kp.num_kb + splits - 1) / splits;
  kp.out = d.out;
  kp.ldc = d.ldc;
  kp.out_f32 = d.out_f32;
  kp.accumulate_out = d.accumulate_out;
  kp.bias = d.bias;
  kp.stats = d.stats;
  kp.split_stride = d.split_stride;
  kp.remap = d.remap;
  kp.rP = d.rP;
  kp.rQ = d.rQ;
  kp.rH = d.rH;
  kp.rW = d.rW;
  kp.rsh = d.rsh;
  kp.rsw = d.rsw;
  const int m_tiles = gemm_m_tiles(d);
  const int n_tiles = (d.N + bn - 1) / bn;
  switch (bn) {
    case 64: return launch_bn<64>(kp, m_tiles, n_tiles, splits, stream);
    case 128: return launch_bn<128>(kp, m_tiles, n_tiles, splits, stream);
    default: return launch_bn<256>(kp, m_tiles, n_tiles, splits, stream);
  }
}

}  // namespace rfk
