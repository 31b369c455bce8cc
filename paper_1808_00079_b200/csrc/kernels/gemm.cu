// Warp-specialised tcgen05 GEMM / implicit-GEMM convolution for sm_100a.
//
//   warp 0      TMA producer (one elected lane): A and B tiles -> smem ring
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..9  epilogue: TMEM -> registers -> global, optional fused
//               per-column statistics (BatchNorm sum / sum of squares);
//               two warps per TMEM lane quarter, alternating 32-column chunks
//
// Tiles: BLOCK_M = 128 output rows, BLOCK_N in {64, 128, 256}, BLOCK_K = 64
// (one 128-byte swizzle row of bf16).  Operands are staged with TMA in
// 128-byte-swizzled layouts, K-major or MN-major, and read by tcgen05.mma
// straight from shared memory; the fp32 accumulator lives in TMEM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>

#include "kernels/kernels.h"
#include "kernels/launch.cuh"
#include "kernels/ptx.cuh"

// Timing-experiment switches (KParams::experiment) exist only in tuning
// builds: as runtime branches in the MMA and epilogue loops they cost the
// production kernel measurable time.
#ifndef RFK_GEMM_TUNING
#define RFK_GEMM_TUNING 0
#endif

namespace rfk {

namespace {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kTileA = kBlockM * kBlockK * 2;  // 16 KB

struct alignas(64) KParams {
  CUtensorMap ta;  // 64-byte aligned, must be first
  CUtensorMap tb;
  CUtensorMap tc;  // output {N, M, splits}: 32x32 bf16 or 16x32 fp32 boxes, SWIZZLE_64B
  CUtensorMap tc2;  // second bf16 output of the fused BN apply (same geometry)
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
  int stats_acc;
  long split_stride;
  int remap, rP, rQ, rH, rW, rsh, rsw;
  int b_taps;  // WeightTapsMN: filter taps R*S
  int b_tap_base, b_tap_dr, b_tap_ds;  // weight tap of A tap (r, s): base - r*dr - s*ds
  int out_mode;  // 0 generic stores, 1 TMA store, 2 TMA reduce-add (accumulate_out)
  int stages;  // smem ring depth in stages (of kps K blocks each)
  int kps;     // K blocks per ring stage (1 or 2; 1 for CTA pairs)
  int m_tiles, n_tiles, splits;  // persistent tile space
  // fused BatchNorm apply (re-forward): out2 = [relu](bf16(D) * scale + shift)
  const float* bn_scale;
  const float* bn_shift;
  int bn_relu, fuse_bn;
  // BN backward statistics in the epilogue (stats_bwd): the output is dout of
  // a BN+ReLU's output (stored as is); the statistics rows hold sum g and
  // sum g*(y - mean) per column, g = dout * [y*scale+shift > 0].
  // replay: no GEMM -- the epilogue re-reads the stored output instead of TMEM
  // (same tiles, same CTAs, same arithmetic: bit-identical rows).
  int stats_bwd, replay;
  const __nv_bfloat16* bs_y;
  long bs_ldy;
  const float* bs_mean;
  const float* bs_scale;
  const float* bs_shift;
  unsigned long long* dbg;  // tuning only: per-tile timeline of CTA 0 (RFK_GEMM_DBG=1)
  int experiment;  // tuning only (builds with RFK_GEMM_TUNING=1): 2 drop the output, 3 also skip TMEM
                  // loads, 4 also skip the MMAs, 5 skip the statistics smem reads, 6 skip the statistics
                  // accumulation, 7 no operand loads (MMAs + epilogue), 8 = 7 without the MMAs, 9 = 8 without
                  // TMEM loads and output (the barrier pipeline alone)
};

template <int BN, bool PAIR = false>
struct Cfg {
  // a CTA of a pair stages half of the B tile
  static constexpr int kTileB = (PAIR ? BN / 2 : BN) * kBlockK * 2;
  static constexpr int kStage = kTileA + kTileB;
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  // epilogue staging: per warp, 1 or 2 buffers of one 32-row x 64-byte box
  static constexpr int kStgBufs = BN == 256 ? 1 : 2;
  static constexpr int kStaging = kEpiWarps * kStgBufs * 2048;
  static constexpr int kStats = kEpiWarps * 2 * (BN / 2) * 4;  // per-warp sums of the warp's own columns
  // as deep a TMA ring as the 227 KB of dynamic shared memory allows
  static constexpr int kSmemMax = 232448;
  static constexpr int kStages = (kSmemMax - kStaging - kStats - 1024 - 256) / kStage;
  static_assert(kStages >= 3, "ring too shallow");
  static constexpr int kSmem = kStages * kStage + kStaging + kStats + 1024 /*align*/ + 256;
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

// Persistent tile loop: CTA b processes tiles b, b + grid, ...; tile t ->
// (m tile fastest, then n tile, then split).  Two TMEM accumulators let the
// epilogue of tile i drain while the MMA warp already accumulates tile i+1,
// and the TMA warp streams K blocks across tile boundaries.
struct TileCoord {
  int m0, n0, z, kb_begin, kb_end;
};

// A CTA pair (PAIR) computes the 256 x BN tile made of M tiles 2i and 2i + 1:
// unit t -> (M tile pair fastest, then n tile, then split), and the CTA of
// cluster rank r drains M tile 2i + r (past the last M tile when m_tiles is
// odd: its A rows load as zeros and nothing is stored).
template <bool PAIR>
__device__ __forceinline__ TileCoord tile_coord(const KParams& p, int t, int BN, int rank) {
  TileCoord c;
  const int mu = PAIR ? (p.m_tiles + 1) >> 1 : p.m_tiles;
  const int mt = PAIR ? 2 * (t % mu) + rank : t % mu;
  const int rest = t / mu;
  c.m0 = mt * kBlockM;
  c.n0 = (rest % p.n_tiles) * BN;
  c.z = rest / p.n_tiles;
  c.kb_begin = c.z * p.kb_per_split;
  c.kb_end = min(p.num_kb, c.kb_begin + p.kb_per_split);
  return c;
}

// Stage one 32-row x 64-byte box (lane = row) in 64B-swizzled smem and hand
// it to the TMA unit; the buffer was last used two boxes ago.
template <int NBUF>
__device__ __forceinline__ void epi_tma_out(const KParams& p, uint8_t* b, const uint32_t (&w)[16], uint32_t lane,
                                            int mode, int cx, int my, int z) {
  if (lane == 0) bulk_wait_read<NBUF - 1>();
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t sw = (uint32_t)j ^ ((lane >> 1) & 3u);  // SWIZZLE_64B
    *reinterpret_cast<uint4*>(b + lane * 64 + sw * 16) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (mode == 2)
      tma_reduce_add_3d(&p.tc, b, cx, my, z);
    else if (mode == 3)
      tma_store_3d(&p.tc2, b, cx, my, z);
    else
      tma_store_3d(&p.tc, b, cx, my, z);
    bulk_commit();
  }
}

// EXT: BN-backward statistics / replay epilogue variants.
// PAIR: launched as 2-CTA clusters running M = 256 tiles with cta_group::2
// MMAs issued by the rank-0 CTA.  Each CTA stages its own 128 A rows and half
// of the B columns, so per SM the shared-memory traffic of a K block (TMA
// writes + MMA reads) drops from A + B to A + B/2 -- the 1-SM kernel is bound
// by it.  Each CTA's epilogue drains its own TMEM (its 128 rows, all BN
// columns); the accumulator is released once both epilogues arrived on the
// leader's barrier.
//
// RES: B resident -- every CTA uses the same B (one n tile, no split) and all
// of it sits in shared memory beside an A-only ring: loaded once per CTA.  A
// separate instance, so the other variants keep their code and registers.
//
// EPI: 0 = every epilogue path; 1 = only the common one -- bf16 output through
// TMA store / TMA reduce-add, optional statistics; 2 = only fp32 output
// through TMA (split-K partials); 3 = 1 plus the fused BN apply (re-forward);
// 4 = only bf16 generic (remapped / unaligned) stores.  No bias compiled into
// 1-4, no generic stores into 1-3.
template <int BN, bool EXT, bool PAIR, bool RES = false, int EPI = 0>
__global__ void __launch_bounds__(kThreads, 1) gemm_kernel(const __grid_constant__ KParams p) {
  constexpr bool SIMPLE = EPI != 0;
  using C = Cfg<BN, PAIR>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by pointer arithmetic on the shared array itself, so
  // every derived pointer keeps the shared address space (LDS/STS, not
  // generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nst = p.stages;
  // K blocks per ring stage: each full / empty barrier hand-off costs the
  // single-thread producer and MMA loops ~300-400 cycles (measured:
  // tools/mma_micro.cu ring_bench), so narrow tiles take two 64-wide K blocks
  // per hand-off
  const int kps = PAIR ? 1 : p.kps;
  // ring slots (nst stages x kps; A + B, A only with RES), [resident B],
  // epilogue staging, column sums, barriers
  constexpr int kStageBytes = RES ? kTileA : C::kStage;
  uint8_t* b_base = smem + nst * kps * kStageBytes;
  uint8_t* stage_buf = RES ? b_base + p.num_kb * C::kTileB : b_base;  // epilogue staging, then the column sums
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_buf + C::kStaging + C::kStats);
  uint64_t* empty = full + nst;
  uint64_t* acc_full = empty + nst;   // [2] MMA -> epilogue
  uint64_t* acc_empty = acc_full + 2; // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  uint64_t* b_full = reinterpret_cast<uint64_t*>(tmem_slot + 2);  // RES: B landed

  const uint32_t warp = warp_id();
  const int ex = RFK_GEMM_TUNING ? p.experiment : 0;
  // persistent unit loop: CTA (pair) t0 takes units t0, t0 + tstep, ...
  const int rank = PAIR ? (int)cluster_ctarank() : 0;
  const int t0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int tstep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int total = (PAIR ? (p.m_tiles + 1) >> 1 : p.m_tiles) * p.n_tiles * p.splits;

  if (warp == 0 && elect_one()) {
    if (!(EXT && p.replay)) {
      tma_prefetch(&p.ta);
      tma_prefetch(&p.tb);
    }
    if (p.out_mode) tma_prefetch(&p.tc);
    if (p.fuse_bn) tma_prefetch(&p.tc2);
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    if (RES) mbar_init(b_full, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], PAIR ? 2 * kEpiWarps : kEpiWarps);  // one arrive per epilogue warp (of both CTAs)
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR)
      tmem_alloc_pair<2 * C::kTmemCols>(tmem_slot);
    else
      tmem_alloc<2 * C::kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // the leader's barriers exist before the peer's loads signal them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // everything above (barrier init, TMEM allocation, descriptor prefetch)
  // overlaps the previous kernel's tail under programmatic dependent launch
  pdl_enter();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one() && !(EXT && p.replay)) {
      int stage = 0;
      uint32_t phase = 0;
      // this CTA's B columns: all BN, or (pair) the half n0 + rank * BN/2
      constexpr int BNB = PAIR ? BN / 2 : BN;
      // the loads of both CTAs of a pair complete on the leader's full barrier
      auto ld2 = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
        if (PAIR)
          tma_load_2d_pair(dst, m, mapa_u32(smem_u32(bar), 0), c0, c1);
        else
          tma_load_2d(dst, m, bar, c0, c1);
      };
      auto ld3 = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
        if (PAIR)
          tma_load_3d_pair(dst, m, mapa_u32(smem_u32(bar), 0), c0, c1, c2);
        else
          tma_load_3d(dst, m, bar, c0, c1, c2);
      };
      auto ldi = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c, int w, int h, int n, uint16_t s,
                     uint16_t r) {
        if (PAIR)
          tma_load_im2col_pair(dst, m, mapa_u32(smem_u32(bar), 0), c, w, h, n, s, r);
        else
          tma_load_im2col(dst, m, bar, c, w, h, n, s, r);
      };
      if constexpr (RES) {
        // the whole B once (one n tile, no split: every tile of this CTA uses it)
        if (RFK_GEMM_TUNING && ex >= 7 && ex <= 9) {
          if (t0 < total) mbar_arrive(b_full);
        } else if (t0 < total) {
          mbar_arrive_expect_tx(b_full, (uint32_t)(p.num_kb * C::kTileB));
          for (int kb = 0; kb < p.num_kb; ++kb) {
            uint8_t* sb = b_base + kb * C::kTileB;
            switch (p.b_kind) {
              case (int)Operand::KMajor2D:
                tma_load_2d(sb, &p.tb, b_full, kb * kBlockK, 0);
                break;
              case (int)Operand::MNMajor2D:
#pragma unroll
                for (int j = 0; j < BN / 64; ++j) tma_load_2d(sb + j * 8192, &p.tb, b_full, 64 * j, kb * kBlockK);
                break;
              default: {  // WeightTapsMN
                const int tap = kb / p.g_cblocks, cb = kb - tap * p.g_cblocks;
                const int tr = tap / p.g_S, ts = tap - tr * p.g_S;
                const int ftap = p.b_tap_base - tr * p.b_tap_dr - ts * p.b_tap_ds;
#pragma unroll
                for (int j = 0; j < BN / 64; ++j) tma_load_3d(sb + j * 8192, &p.tb, b_full, 64 * j, ftap, cb * 64);
              }
            }
          }
        }
      }
      int plocal = 0;
      for (int t = t0; t < total; t += tstep, ++plocal) {
        const TileCoord tc = tile_coord<PAIR>(p, t, BN, rank);
        const int n0b = tc.n0 + rank * BNB;
        if (RFK_GEMM_TUNING && p.dbg && blockIdx.x == 0 && plocal < 32) p.dbg[plocal * 8 + 5] = global_ns();
        int aw = 0, ah = 0, an = 0;
        if (p.a_kind == (int)Operand::Im2colK) pixel_base(p, tc.m0, aw, ah, an);
        // K block -> (filter tap (r, s), channel block cb), advanced
        // incrementally (no integer divisions per K block)
        int kcb = 0, ks = 0, kr = 0;
        if (p.a_kind == (int)Operand::Im2colK) {
          const int tap = tc.kb_begin / p.g_cblocks;
          kcb = tc.kb_begin - tap * p.g_cblocks;
          kr = tap / p.g_S;
          ks = tap - kr * p.g_S;
        }
        for (int kb0 = tc.kb_begin; kb0 < tc.kb_end; kb0 += kps) {
          const int nk = min(kps, tc.kb_end - kb0);
          mbar_wait(&empty[stage], phase ^ 1);
          if (RFK_GEMM_TUNING && ex >= 7 && ex <= 9) {  // timing only: no operand loads
            mbar_arrive(&full[stage]);
            if (++stage == nst) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], (uint32_t)nk * (PAIR ? 2 * C::kStage : kStageBytes));
          for (int j = 0; j < nk; ++j) {
            const int kb = kb0 + j;
            uint8_t* sa = smem + (stage * kps + j) * kStageBytes;
            uint8_t* sb = sa + kTileA;
            switch (p.a_kind) {
              case (int)Operand::KMajor2D:
                ld2(sa, &p.ta, &full[stage], kb * kBlockK, tc.m0);
                break;
              case (int)Operand::MNMajor2D:
                ld2(sa, &p.ta, &full[stage], tc.m0, kb * kBlockK);
                ld2(sa + kTileA / 2, &p.ta, &full[stage], tc.m0 + 64, kb * kBlockK);
                break;
              default:  // Im2colK: K block -> (tap, channel block)
                ldi(sa, &p.ta, &full[stage], kcb * 64, aw, ah, an, (uint16_t)ks, (uint16_t)kr);
            }
            if (!RES) switch (p.b_kind) {
              case (int)Operand::KMajor2D:  // box of BNB rows
                ld2(sb, &p.tb, &full[stage], kb * kBlockK, n0b);
                break;
              case (int)Operand::MNMajor2D:
#pragma unroll
                for (int jj = 0; jj < BNB / 64; ++jj)
                  ld2(sb + jj * 8192, &p.tb, &full[stage], n0b + 64 * jj, kb * kBlockK);
                break;
              case (int)Operand::WeightTapsMN: {  // K block = (tap of the im2col A, Cout block), flipped
                const int ftap = p.b_tap_base - kr * p.b_tap_dr - ks * p.b_tap_ds;
#pragma unroll
                for (int jj = 0; jj < BNB / 64; ++jj)
                  ld3(sb + jj * 8192, &p.tb, &full[stage], n0b + 64 * jj, ftap, kcb * 64);
                break;
              }
              default: {  // Im2colMN: K block = 64 output pixels, MN = (tap, channel)
                int bw, bh, bn;
                pixel_base(p, kb * kBlockK, bw, bh, bn);
#pragma unroll
                for (int jj = 0; jj < BNB / 64; ++jj) {
                  const int nb = n0b / 64 + jj;
                  const int tap = nb / p.g_cblocks, cb = nb - tap * p.g_cblocks;
                  const int r = tap / p.g_S, s = tap - r * p.g_S;
                  ldi(sb + jj * 8192, &p.tb, &full[stage], cb * 64, bw, bh, bn, (uint16_t)s, (uint16_t)r);
                }
              }
            }
            if (++kcb == p.g_cblocks) {
              kcb = 0;
              if (++ks == p.g_S) {
                ks = 0;
                ++kr;
              }
            }
          }
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (PAIR) {
        // the leader's last MMA commits arrive on this CTA's empty barriers:
        // wait for them before the CTA may exit
        for (int i = 0; i < nst; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const bool a_mn = p.a_kind == (int)Operand::MNMajor2D;
    const bool b_mn = p.b_kind == (int)Operand::MNMajor2D || p.b_kind == (int)Operand::Im2colMN ||
                      p.b_kind == (int)Operand::WeightTapsMN;
    const uint32_t idesc = umma_idesc_bf16(PAIR ? 2 * kBlockM : kBlockM, BN, a_mn, b_mn);
    // Descriptors as (low word = start address >> 4 | LBO, high word = SBO |
    // version | swizzle): per K block only the start advances, by the stage
    // offset, and per 16-wide K step by 32 bytes (K-major) or 2048 bytes
    // (MN-major), so the issue loop is a handful of uniform adds.
    const uint64_t a_d0 = a_mn ? umma_desc_sw128(smem_u32(smem), 8192, 1024) : umma_desc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t b_d0 = b_mn ? umma_desc_sw128(smem_u32(RES ? b_base : smem + kTileA), 8192, 1024)
                               : umma_desc_sw128(smem_u32(RES ? b_base : smem + kTileA), 16, 1024);
    const uint32_t a_lo0 = (uint32_t)a_d0, a_hi = (uint32_t)(a_d0 >> 32);
    const uint32_t b_lo0 = (uint32_t)b_d0, b_hi = (uint32_t)(b_d0 >> 32);
    const uint32_t a_kstep = a_mn ? (2048u >> 4) : (32u >> 4);
    const uint32_t b_kstep = b_mn ? (2048u >> 4) : (32u >> 4);
    constexpr uint32_t kStageStep = (uint32_t)kStageBytes >> 4;
    constexpr uint32_t kResStep = (uint32_t)C::kTileB >> 4;
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    if (RES && t0 < total) mbar_wait(b_full, 0);
    // (pair: the rank-1 CTA issues nothing; the leader's MMAs fill both TMEMs)
    for (int t = t0; t < ((EXT && p.replay) || rank != 0 ? 0 : total); t += tstep, ++local) {
      const TileCoord tc = tile_coord<PAIR>(p, t, BN, rank);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);  // epilogue(s) drained this accumulator
      tc_fence_after();
      if (RFK_GEMM_TUNING && p.dbg && blockIdx.x == 0 && local < 32 && lane_id() == 0) p.dbg[local * 8 + 0] = global_ns();
      const uint32_t d_tmem = tmem + (uint32_t)(acc * C::kTmemCols);
      if (tc.kb_end <= tc.kb_begin) {
        if (elect_one()) {  // empty split: nothing to accumulate
          mbar_arrive(&acc_full[acc]);
          if (PAIR) mbar_arrive_cluster(mapa_u32(smem_u32(&acc_full[acc]), 1));
        }
        __syncwarp();
        continue;
      }
      for (int kb0 = tc.kb_begin; kb0 < tc.kb_end; kb0 += kps) {
        const int nk = min(kps, tc.kb_end - kb0);
        const int kb = kb0 + nk - 1;  // the stage's last K block
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          for (int j = 0; j < nk; ++j) {
            const uint32_t a_lo = a_lo0 + (uint32_t)(stage * kps + j) * kStageStep;
            const uint32_t b_lo =
                b_lo0 + (RES ? (uint32_t)(kb0 + j) * kResStep : (uint32_t)(stage * kps + j) * kStageStep);
#pragma unroll
            for (int kk = 0; kk < ((ex == 4 || ex == 8 || ex == 9) ? 0 : kBlockK / 16); ++kk) {
              const uint64_t da = ((uint64_t)a_hi << 32) | (a_lo + (uint32_t)kk * a_kstep);
              const uint64_t db = ((uint64_t)b_hi << 32) | (b_lo + (uint32_t)kk * b_kstep);
              const uint32_t accum = (kb0 + j > tc.kb_begin || kk > 0) ? 1u : 0u;
              if (PAIR)
                umma_bf16_pair(d_tmem, da, db, idesc, accum);
              else
                umma_bf16(d_tmem, da, db, idesc, accum);
            }
          }
          if (RFK_GEMM_TUNING && p.dbg && blockIdx.x == 0 && local < 32 && kb + 1 == tc.kb_end) p.dbg[local * 8 + 1] = global_ns();
          if (PAIR) {
            umma_commit_pair(&empty[stage]);
            if (kb + 1 == tc.kb_end) umma_commit_pair(&acc_full[acc]);
          } else {
            umma_commit(&empty[stage]);
            if (kb + 1 == tc.kb_end) umma_commit(&acc_full[acc]);
          }
        }
        __syncwarp();
        if (++stage == nst) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..9)
    // TMEM -> registers (32 columns at a time) -> [bias] -> [column statistics]
    // -> 64-byte-swizzled smem staging -> TMA store / TMA reduce-add of a
    // 32-row box.  Warp w reads TMEM lanes 32 * (w % 4) (the hardware's lane
    // quarter rule); the two warps of a quarter take alternating 32-column
    // chunks, so eight warps drain an accumulator in parallel.
    const uint32_t quarter = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const uint32_t ew = warp - 2;  // epilogue warp index 0..7
    const uint32_t lane = lane_id();
    constexpr int NB = C::kStgBufs;
    uint8_t* stg = stage_buf + ew * (NB * 2048);
    // Fused BN statistics: each warp keeps its own per-column sums in smem
    // for the columns it owns (lane l owns column pair 2 (l & 15) of a chunk,
    // so no synchronisation per chunk); when the CTA moves to another column
    // block the eight warps' sums are combined in a fixed order and written
    // once as this CTA's row of stats[gridDim][2][N].  The finalize then sums
    // ~148 rows instead of one per M tile.  Rows of column blocks a CTA never
    // touches stay zero (workspace zeroed once; the tile -> CTA mapping is the
    // same every launch).
    constexpr int HB = BN / 2;  // columns owned by one warp
    float* wsum = reinterpret_cast<float*>(stage_buf + C::kStaging);  // [8 warps][2][HB]
    float* my_sum = wsum + ew * 2 * HB;
    const int mode = p.out_mode;
    const bool f32 = EPI == 2 || (EPI == 0 && p.out_f32);
    const float* bias = SIMPLE ? nullptr : p.bias;
    const bool fuse = EPI == 3 || (EPI == 0 && p.fuse_bn);
    const bool tma = EPI == 4 ? false : (SIMPLE || mode != 0);
    int buf = 0;
    auto tma_out = [&](const uint32_t(&w)[16], int cx, int my, int z) {
      epi_tma_out<NB>(p, stg + buf * 2048, w, lane, mode, cx, my, z);
      if (NB == 2) buf ^= 1;
    };
    int cur_nt = -1;
    auto flush_stats = [&](int nt) {
      asm volatile("bar.sync 1, 256;" ::: "memory");
      float* row = p.stats + (long)blockIdx.x * 2 * p.N;
      for (int c = (int)(ew * 32 + lane); c < BN; c += 256) {
        const int j = c >> 5, h = j & 1, lc = ((j >> 1) << 5) + (c & 31);
        float s = 0.f, q = 0.f;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          // warp of (half h, quarter qq): ew = 4 h + ((qq + 2) & 3)
          float* ws = wsum + (4 * h + ((qq + 2) & 3)) * 2 * HB;
          s += ws[lc];
          q += ws[HB + lc];
        }
        const int col = nt * BN + c;
        if (col < p.N) {
          if (p.stats_acc) s += row[col], q += row[p.N + col];  // earlier chunks of M first
          row[col] = s;
          row[p.N + col] = q;
        }
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
      for (int c = (int)lane; c < 2 * HB; c += 32) my_sum[c] = 0.f;
      __syncwarp();
    };
    if (p.stats) {
      for (int c = (int)lane; c < 2 * HB; c += 32) my_sum[c] = 0.f;
      __syncwarp();
    }
    int local = 0;
    for (int t = t0; t < total; t += tstep, ++local) {
      const TileCoord tc = tile_coord<PAIR>(p, t, BN, rank);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const bool empty_k = tc.kb_end <= tc.kb_begin;
      if (p.stats && tc.n0 / BN != cur_nt) {
        if (cur_nt >= 0) flush_stats(cur_nt);
        cur_nt = tc.n0 / BN;
      }
      if (!(EXT && p.replay)) {
        mbar_wait(&acc_full[acc], acc_phase);
        tc_fence_after();
      }
      if (RFK_GEMM_TUNING && p.dbg && blockIdx.x == 0 && local < 32 && ew == 0 && lane == 0) p.dbg[local * 8 + 2] = global_ns();
      const int my = tc.m0 + (int)(quarter * 32);
      const int m = my + (int)lane;
      const bool row_ok = m < p.M;
#pragma unroll 1
      for (int c0 = (int)half * 32; c0 < BN; c0 += 64) {
        // BN-backward statistics: this chunk's BN-input values (lane: column
        // pair 2 (lane & 15), even / odd rows) are loaded first, so their
        // latency overlaps the TMEM load and the output staging
        uint32_t yv[16];
        float2 bmu = make_float2(0.f, 0.f), bsc = bmu, bsh = bmu;
        if (EXT && p.stats_bwd) {
          const int c = tc.n0 + c0 + 2 * (int)(lane & 15);
          const bool col_ok = c < p.N;
          if (col_ok) {
            bmu = __ldg(reinterpret_cast<const float2*>(p.bs_mean + c));
            bsc = __ldg(reinterpret_cast<const float2*>(p.bs_scale + c));
            bsh = __ldg(reinterpret_cast<const float2*>(p.bs_shift + c));
          }
#pragma unroll
          for (int rr = 0; rr < 16; ++rr) {
            const int mr = my + 2 * rr + (int)(lane >> 4);
            yv[rr] = (col_ok && mr < p.M) ? __ldg(reinterpret_cast<const unsigned int*>(p.bs_y + (long)mr * p.bs_ldy + c))
                                          : 0u;
          }
        }
        uint32_t r[32];
        if (EXT && p.replay) {
          // the stored bf16 output of this lane's row, 32 columns
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 u = make_uint4(0u, 0u, 0u, 0u);
            if (row_ok && tc.n0 + c0 + 8 * j < p.N)
              u = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(p.out) +
                                                       (long)m * p.ldc + tc.n0 + c0 + 8 * j));
            const uint32_t uw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              r[8 * j + 2 * e] = uw[e] << 16;              // low bf16 -> fp32 bits
              r[8 * j + 2 * e + 1] = uw[e] & 0xffff0000u;  // high bf16 -> fp32 bits
            }
          }
        } else if (!empty_k && (ex < 3 || ex > 4) && ex != 9) {
          tmem_ld32(tmem + (uint32_t)(acc * C::kTmemCols) + ((quarter * 32u) << 16) + (uint32_t)c0, r);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        if (RFK_GEMM_TUNING && p.dbg && blockIdx.x == 0 && local < 32 && ew == 0 && lane == 0 && c0 < 64) p.dbg[local * 8 + 3] = global_ns();
        if (c0 + 64 >= BN && !(EXT && p.replay)) {
          // this warp's last chunk of the accumulator is in registers: hand it back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR && rank != 0)
              mbar_arrive_cluster(mapa_u32(smem_u32(&acc_empty[acc]), 0));
            else
              mbar_arrive(&acc_empty[acc]);
          }
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        const int col0 = tc.n0 + c0;
        if (col0 >= p.N || (ex >= 2 && ex <= 4) || ex == 9) continue;  // warp-uniform
        const bool full_cols = col0 + 32 <= p.N;
        if (bias) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += (col0 + i < p.N) ? __ldg(bias + col0 + i) : 0.f;
        }
        if (f32) {
          if (mode != 0) {  // two 16-column fp32 boxes
            uint32_t w[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(v[i]);
            tma_out(w, col0, my, tc.z);
            if (col0 + 16 < p.N) {
#pragma unroll
              for (int i = 0; i < 16; ++i) w[i] = __float_as_uint(v[16 + i]);
              tma_out(w, col0 + 16, my, tc.z);
            }
          } else if (row_ok) {
            float* dst = reinterpret_cast<float*>(p.out) + (long)tc.z * p.split_stride + (long)m * p.ldc + col0;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.N) dst[i] = p.accumulate_out ? dst[i] + v[i] : v[i];
          }
          continue;
        }
        // bf16: rows past M are staged as zeros (TMA clips them on store; the
        // statistics below then need no row mask)
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) w[i] = row_ok ? pack_bf16(v[2 * i], v[2 * i + 1]) : 0u;
        const uint8_t* sbuf;
        if (EXT && p.replay) {
          // statistics only: stage (same layout as the store paths), no write
          uint8_t* gb = stg;
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t sw = (uint32_t)j ^ ((lane >> 1) & 3u);
            *reinterpret_cast<uint4*>(gb + lane * 64 + sw * 16) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
          }
          __syncwarp();
          sbuf = gb;
        } else if (tma) {
          sbuf = stg + buf * 2048;
          tma_out(w, col0, my, tc.z);
          if (fuse) {
            // the BN that consumes this conv, applied to exactly the bf16
            // values just stored (same expression as bn_apply_kernel)
            uint32_t w2[16];
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const int c = col0 + 2 * i;
              const float4 sc = __ldg(reinterpret_cast<const float4*>(p.bn_scale + c));
              const float4 sh = __ldg(reinterpret_cast<const float4*>(p.bn_shift + c));
              const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
              const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i + 1]));
              float o0 = fmaf(a.x, sc.x, sh.x), o1 = fmaf(a.y, sc.y, sh.y);
              float o2 = fmaf(b.x, sc.z, sh.z), o3 = fmaf(b.y, sc.w, sh.w);
              if (p.bn_relu) {
                o0 = fmaxf(o0, 0.f);
                o1 = fmaxf(o1, 0.f);
                o2 = fmaxf(o2, 0.f);
                o3 = fmaxf(o3, 0.f);
              }
              w2[i] = row_ok ? pack_bf16(o0, o1) : 0u;
              w2[i + 1] = row_ok ? pack_bf16(o2, o3) : 0u;
            }
            epi_tma_out<C::kStgBufs>(p, stg + buf * 2048, w2, lane, 3, col0, my, tc.z);
            if (C::kStgBufs == 2) buf ^= 1;
          }
        } else {
          // generic: stage, then write whole 64-byte row segments with 4
          // lanes per row (8 rows per instruction)
          uint8_t* gb = stg;
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t sw = (uint32_t)j ^ ((lane >> 1) & 3u);
            *reinterpret_cast<uint4*>(gb + lane * 64 + sw * 16) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
          }
          __syncwarp();
          // four 8-row passes: addresses and (accumulating) the previous
          // values of all four are loaded before any store, so the scattered
          // read-modify-write of a remapped output costs one memory round
          // trip per chunk, not four
          const uint32_t chunk = lane & 3;
          __nv_bfloat16* dsts[4];
          uint4 vals[4], prevs[4];
          bool oks[4], fulls[4];
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const uint32_t row = it * 8 + (lane >> 2);
            vals[it] = *reinterpret_cast<const uint4*>(gb + row * 64 + ((chunk ^ ((row >> 1) & 3u)) * 16));
            const int mr = my + (int)row;
            oks[it] = mr < p.M && (full_cols || col0 + (int)chunk * 8 < p.N);
            fulls[it] = full_cols || col0 + (int)chunk * 8 + 8 <= p.N;
            long orow = mr;
            if (p.remap) {
              const int q = mr % p.rQ, tt = mr / p.rQ, pp = tt % p.rP, nn = tt / p.rP;
              orow = (long)nn * p.rH * p.rW + (long)(pp * p.rsh) * p.rW + (long)q * p.rsw;
            }
            dsts[it] = reinterpret_cast<__nv_bfloat16*>(p.out) + (long)tc.z * p.split_stride + orow * p.ldc + col0 +
                       chunk * 8;
            if (p.accumulate_out && oks[it] && fulls[it]) prevs[it] = *reinterpret_cast<const uint4*>(dsts[it]);
          }
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            if (!oks[it]) continue;
            __nv_bfloat16* dst = dsts[it];
            const uint4 val = vals[it];
            const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&val);
            if (fulls[it]) {
              uint4 o = val;
              if (p.accumulate_out) {
                const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&val);
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&prevs[it]);
                __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 fa = __bfloat1622float2(a2[e]), fb = __bfloat1622float2(b2[e]);
                  o2[e] = __floats2bfloat162_rn(fa.x + fb.x, fa.y + fb.y);
                }
              }
              *reinterpret_cast<uint4*>(dst) = o;
            } else {
              for (int e = 0; e < 8 && col0 + (int)chunk * 8 + e < p.N; ++e)
                dst[e] = p.accumulate_out ? __float2bfloat16_rn(__bfloat162float(dst[e]) + __bfloat162float(vb[e]))
                                          : vb[e];
            }
          }
          sbuf = gb;
        }
        if (p.stats) {
          // Column sums of the staged (bf16-rounded: exactly what the
          // BatchNorm reads back) 32 x 32 tile: lane l sums the column pair
          // 2 (l & 15) over the even (l < 16) or odd rows, then the two row
          // halves combine with one shuffle.  Even/odd rows sit in opposite
          // 64-byte halves of the bank space, so the reads are conflict-free.
          const uint32_t cp = lane & 15, par = lane >> 4;
          float s0 = 0.f, s1 = 0.f, q0 = 0.f, q1 = 0.f;
          if (EXT && p.stats_bwd) {
            // sum g and sum g * (y - mean) over the chunk's rows (rows past M
            // and columns past N were staged as g = 0)
            const float2 mu = bmu, sc = bsc, sh = bsh;
#pragma unroll
            for (int rr = 0; rr < 16; ++rr) {
              const uint32_t row = 2 * rr + par;
              const uint32_t off = row * 64 + (((cp >> 2) ^ ((row >> 1) & 3u)) * 16) + (cp & 3) * 4;
              float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sbuf + off));
              const float ylo = __uint_as_float(yv[rr] << 16), yhi = __uint_as_float(yv[rr] & 0xffff0000u);
              // g = dout * [y * scale + shift > 0]: the BN+ReLU backward's
              // mask, same expression as bn_bwd_apply MODE 1
              if (!(fmaf(ylo, sc.x, sh.x) > 0.f)) g.x = 0.f;
              if (!(fmaf(yhi, sc.y, sh.y) > 0.f)) g.y = 0.f;
              s0 += g.x;
              s1 += g.y;
              q0 = fmaf(g.x, ylo - mu.x, q0);
              q1 = fmaf(g.y, yhi - mu.y, q1);
            }
          } else {
#pragma unroll
          for (int rr = 0; rr < (ex == 5 ? 0 : 16); ++rr) {
            const uint32_t row = 2 * rr + par;
            const uint32_t off = row * 64 + (((cp >> 2) ^ ((row >> 1) & 3u)) * 16) + (cp & 3) * 4;
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sbuf + off));
            s0 += f.x;
            s1 += f.y;
            q0 = fmaf(f.x, f.x, q0);
            q1 = fmaf(f.y, f.y, q1);
          }
          }
          s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
          q0 += __shfl_xor_sync(0xffffffffu, q0, 16);
          q1 += __shfl_xor_sync(0xffffffffu, q1, 16);
          if (lane < 16 && ex != 6) {
            const int lc = ((c0 >> 6) << 5) + 2 * (int)lane;  // this warp's local column
            my_sum[lc] += s0;
            my_sum[lc + 1] += s1;
            my_sum[HB + lc] += q0;
            my_sum[HB + lc + 1] += q1;
          }
        }
        __syncwarp();
      }
      if (RFK_GEMM_TUNING && p.dbg && blockIdx.x == 0 && local < 32 && ew == 0 && lane == 0) p.dbg[local * 8 + 4] = global_ns();
    }
    if (p.stats && cur_nt >= 0) flush_stats(cur_nt);
    if (lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync();  // neither CTA leaves (or frees TMEM) while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    if (PAIR)
      tmem_dealloc_pair<2 * C::kTmemCols>(tmem);
    else
      tmem_dealloc<2 * C::kTmemCols>(tmem);
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
  // stride 1: the box spans exactly the Q x P output bases, which also covers
  // asymmetric padding (the sub-pixel dgrad classes pad only the high side)
  if (g.stride_w == 1) upper[0] = g.Q - g.W - g.pad_w;
  if (g.stride_h == 1) upper[1] = g.P - g.H - g.pad_h;
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

// CTA pairs for launches that leave the choice to the engine (desc.pair ==
// 0): RFK_GEMM_PAIR=0 (default) never, 1 where the main loop dominates, 2
// wherever the shapes allow.  Off by default: the training step's GEMMs are
// bound by the operand feed and the epilogue, not the MMA rate, and inside
// the step's graph a 2-CTA cluster also waits for two free SMs of a TPC
// (ResNet-50 step 5.390 ms without pairs, 5.449 ms with the automatic rule).
int pair_mode() {
  static const int m = [] {
    const char* e = std::getenv("RFK_GEMM_PAIR");
    return e == nullptr ? 0 : std::atoi(e);
  }();
  return m;
}

// how many CTA pairs of this kernel can be resident at once (the GPCs need
// not split into SM pairs evenly)
template <int BN>
int pair_max_clusters() {
  static int n = -1;
  if (n < 0) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cfg<BN, true>::kSmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, gemm_kernel<BN, false, true>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    n = c;
    if (std::getenv("RFK_TRACE_PAIR")) std::fprintf(stderr, "rfk: bn=%d pairs resident=%d\n", BN, n);
  }
  return n;
}

template <int BN>
cudaError_t launch_bn_impl(KParams& kp, int m_tiles, int n_tiles, int splits, int max_ctas, bool pair, cudaStream_t st);

// Tuning builds: RFK_GEMM_DBG=1 records CTA 0's per-tile timeline and prints
// it after the (eager, synchronised) launch.
template <int BN>
cudaError_t launch_bn(KParams& kp, int m_tiles, int n_tiles, int splits, int max_ctas, bool pair, cudaStream_t st) {
  static unsigned long long* dbg = nullptr;
  static const bool dbg_on = [] {
    const char* e = std::getenv("RFK_GEMM_DBG");
    return RFK_GEMM_TUNING && e && std::atoi(e) != 0;
  }();
  if (dbg_on && !dbg) cudaMalloc(&dbg, 32 * 8 * sizeof(unsigned long long));
  kp.dbg = dbg_on ? dbg : nullptr;
  if (dbg_on) cudaMemsetAsync(dbg, 0, 32 * 8 * sizeof(unsigned long long), st);
  cudaError_t e = launch_bn_impl<BN>(kp, m_tiles, n_tiles, splits, max_ctas, pair, st);
  if (dbg_on && e == cudaSuccess) {
    unsigned long long h[32 * 8];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, dbg, sizeof(h), cudaMemcpyDeviceToHost);
    unsigned long long t0 = h[5];
    for (int i = 0; i < 8 * 32; ++i)
      if (h[i] && h[i] < t0) t0 = h[i];
    std::printf("gemm dbg BN=%d M=%d N=%d K=%d tiles %d x %d (ns from CTA 0 start): prod_tile mma_acc_free mma_last_kb "
                "epi_acc_full epi_tmem1 epi_done\n", BN, kp.M, kp.N, kp.K, m_tiles, n_tiles);
    for (int l = 0; l < 32 && h[l * 8 + 5]; ++l) {
      auto f = [&](int j) { return h[l * 8 + j] ? (long long)(h[l * 8 + j] - t0) : -1LL; };
      std::printf("  tile %2d: %7lld %7lld %7lld %7lld %7lld %7lld\n", l, f(5), f(0), f(1), f(2), f(3), f(4));
    }
  }
  return e;
}

template <int BN>
cudaError_t launch_bn_impl(KParams& kp, int m_tiles, int n_tiles, int splits, int max_ctas, bool pair, cudaStream_t st) {
  using C = Cfg<BN>;
  using CP = Cfg<BN, true>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e =
        cudaFuncSetAttribute(gemm_kernel<BN, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_kernel<BN, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_kernel<BN, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CP::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_kernel<BN, false, false, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_kernel<BN, true, false, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_kernel<BN, false, false, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_kernel<BN, false, false, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(gemm_kernel<BN, false, false, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               C::kSmem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // persistent grid: one CTA per SM (two TMEM accumulators of BN columns)
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int cap = max_ctas > 0 ? std::min(max_ctas, sms) : sms;
  const long total = (long)(pair ? (m_tiles + 1) / 2 : m_tiles) * n_tiles * splits;  // units (tile pairs)
  int grid;
  if (pair) {
    const int clusters = std::min(pair_max_clusters<BN>(), cap / 2);
    if (clusters <= 0) return cudaErrorInvalidValue;
    grid = 2 * (int)std::min<long>(total, clusters);
  } else {
    grid = (int)std::min<long>(total, cap);
  }
  const int units_grid = pair ? grid / 2 : grid;
  kp.m_tiles = m_tiles;
  kp.n_tiles = n_tiles;
  kp.splits = splits;
  const long kb_per_cta = (long)kp.kb_per_split * ((total + units_grid - 1) / units_grid);
  const int max_stages = pair ? CP::kStages : C::kStages;
  // K blocks per ring stage (RFK_GEMM_KPS overrides): two for tiles whose
  // K block of MMAs is shorter than a barrier hand-off (BN <= 128)
  static const int kps_env = [] {
    const char* e = std::getenv("RFK_GEMM_KPS");
    return e ? std::atoi(e) : 0;
  }();
  // (tuning: 1 off, 2 BN <= 128, 3 every BN, 4 BN = 64 only, 5 where >= 3 stages of 2 fit)
  const int kmode = kps_env > 0 ? kps_env : 2;
  kp.kps = (pair || kp.replay) ? 1
           : (kmode == 3 || (kmode == 2 && BN <= 128) || (kmode == 4 && BN == 64) || (kmode == 5 && max_stages >= 6))
               ? 2
               : 1;
  if (max_stages / kp.kps < 2) kp.kps = 1;
  kp.stages = (int)std::max<long>(2, std::min<long>(max_stages / kp.kps, (kb_per_cta + kp.kps - 1) / kp.kps));
  static const int force_stages = [] {
    const char* e = std::getenv("RFK_GEMM_STAGES");  // tuning experiments only
    return e ? std::atoi(e) : 0;
  }();
  if (force_stages >= 2) kp.stages = std::min(force_stages, max_stages / kp.kps);
  if (kp.replay) kp.stages = 2;  // no operand ring in a statistics replay
  static const int experiment = [] {
    const char* e = std::getenv("RFK_GEMM_EXPERIMENT");  // tuning experiments only
    return e ? std::atoi(e) : 0;
  }();
  kp.experiment = experiment;
  if (experiment == 1 || experiment == 10) kp.out_mode = 0;  // 10: generic stores in the specialised instance
  if (pair) {
    const int smem = kp.stages * CP::kStage + CP::kStaging + CP::kStats + 1024 + 256;
    return launch_k_cluster(gemm_kernel<BN, false, true>, grid, kThreads, smem, st, 2, kp);
  }
  // the common epilogues (RFK_GEMM_SIMPLE=0 turns the specialised instances off)
  static const bool simple_on = [] {
    const char* e = std::getenv("RFK_GEMM_SIMPLE");
    return e == nullptr || std::atoi(e) != 0;
  }();
  const int epi = (simple_on && !kp.replay && !kp.bias && (experiment == 0 || experiment >= 7))
                      ? (kp.out_mode != 0 ? (kp.fuse_bn ? 3 : (kp.out_f32 ? 2 : 1)) : (!kp.out_f32 && !kp.fuse_bn ? 4 : 0))
                      : 0;
  const bool simple = epi == 1;
  // B resident (RFK_GEMM_BRES=0 turns it off): A through TMA im2col, one n
  // tile, no split, several tiles per CTA, and B fits beside an A-only ring of
  // >= 4 stages.  The B bytes a CTA pulls through L2 drop from (tiles x B) to
  // one B: for the N = 64 3x3 convs B is a third of the operand feed that
  // bounds them (tools/gemm_probe.py: 29.4 -> 27.1 us).
  static const bool bres_on = [] {
    const char* e = std::getenv("RFK_GEMM_BRES");
    return e == nullptr || std::atoi(e) != 0;
  }();
  const long b_bytes = (long)kp.num_kb * C::kTileB;
  const long fixed = C::kStaging + C::kStats + 1024 + 256;
  if (bres_on && !kp.replay && kp.a_kind == (int)Operand::Im2colK && kp.b_kind != (int)Operand::Im2colMN &&
      n_tiles == 1 && splits == 1 && total > grid && force_stages < 2 && (experiment == 0 || experiment >= 7) &&
      fixed + b_bytes + 4L * kTileA <= C::kSmemMax) {
    static bool res_configured = false;
    if (!res_configured) {
      cudaError_t e = cudaFuncSetAttribute(gemm_kernel<BN, false, false, true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemMax);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(gemm_kernel<BN, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::kSmemMax);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(gemm_kernel<BN, false, false, true, 1>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemMax);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(gemm_kernel<BN, true, false, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::kSmemMax);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(gemm_kernel<BN, false, false, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::kSmemMax);
      if (e != cudaSuccess) return e;
      res_configured = true;
    }
    const long ring = std::min<long>((C::kSmemMax - fixed - b_bytes) / kTileA, 12);
    if (ring / kp.kps < 2 || (kmode == 5 && ring < 6)) kp.kps = 1;
    kp.stages = (int)std::max<long>(2, std::min<long>(ring / kp.kps, (kb_per_cta + kp.kps - 1) / kp.kps));
    const int smem = (int)(kp.stages * kp.kps * kTileA + b_bytes + fixed);
    if (kp.stats_bwd && simple) return launch_k(gemm_kernel<BN, true, false, true, 1>, grid, kThreads, smem, st, kp);
    if (kp.stats_bwd) return launch_k(gemm_kernel<BN, true, false, true>, grid, kThreads, smem, st, kp);
    if (simple) return launch_k(gemm_kernel<BN, false, false, true, 1>, grid, kThreads, smem, st, kp);
    if (epi == 3) return launch_k(gemm_kernel<BN, false, false, true, 3>, grid, kThreads, smem, st, kp);
    return launch_k(gemm_kernel<BN, false, false, true>, grid, kThreads, smem, st, kp);
  }
  const int smem = kp.stages * kp.kps * C::kStage + C::kStaging + C::kStats + 1024 + 256;
  if (kp.stats_bwd && simple) return launch_k(gemm_kernel<BN, true, false, false, 1>, grid, kThreads, smem, st, kp);
  if (kp.stats_bwd || kp.replay) return launch_k(gemm_kernel<BN, true, false>, grid, kThreads, smem, st, kp);
  if (simple) return launch_k(gemm_kernel<BN, false, false, false, 1>, grid, kThreads, smem, st, kp);
  if (epi == 2) return launch_k(gemm_kernel<BN, false, false, false, 2>, grid, kThreads, smem, st, kp);
  if (epi == 3) return launch_k(gemm_kernel<BN, false, false, false, 3>, grid, kThreads, smem, st, kp);
  if (epi == 4 && !kp.stats_bwd) return launch_k(gemm_kernel<BN, false, false, false, 4>, grid, kThreads, smem, st, kp);
  return launch_k(gemm_kernel<BN, false, false>, grid, kThreads, smem, st, kp);
}

}  // namespace

int gemm_m_tiles(const GemmDesc& d) { return (d.M + kBlockM - 1) / kBlockM; }

int gemm_block_n(const GemmDesc& d) {
  int bn = d.block_n;
  if (bn == 0) {
    // Empirical cost model, fitted to a B200 sweep of every ResNet-50 GEMM
    // shape over tile widths and split counts (tools/gemm_sweep.py):
    //   t(bn) = waves * (k_blocks * a + b)   [us]
    // a = cost of one 64-deep K block of a 128 x bn tile: ~0.5 us whenever A
    // comes through TMA im2col (the im2col load, not the MMA, is the limit,
    // so wider tiles are free work), 0.20 / 0.25 / 0.30 us for plain 2-D
    // tiles; b = per-tile prologue + epilogue, 2.5 / 3.5 / 7 us.
    const long mt = (d.M + kBlockM - 1) / kBlockM;
    const int splits = std::max(1, d.splits);
    long kb;
    if (d.a_kind == Operand::Im2colK)
      kb = (long)d.a_geom.R * d.a_geom.S * ((d.a_geom.C + 63) / 64);
    else
      kb = (d.K + 63) / 64;
    kb = (kb + splits - 1) / splits;
    const bool im2col = d.a_kind == Operand::Im2colK;
    double best = -1;
    for (int cand : {256, 128, 64}) {
      if (cand > 64 && d.N <= cand / 2) continue;
      const long tiles = mt * ((d.N + cand - 1) / cand) * splits;
      const long waves = (tiles + 147) / 148;
      const double a = im2col ? 0.5 : (cand == 64 ? 0.20 : (cand == 128 ? 0.25 : 0.30));
      const double b = cand == 64 ? 2.5 : (cand == 128 ? 3.5 : 7.0);
      const double cost = (double)waves * ((double)kb * a + b);
      if (best < 0 || cost < best) {
        best = cost;
        bn = cand;
      }
    }
  }
  if (d.b_kind == Operand::MNMajor2D || d.b_kind == Operand::Im2colMN || d.b_kind == Operand::WeightTapsMN)
    bn = bn < 64 ? 64 : bn;
  return bn;
}

cudaError_t gemm_launch(const GemmDesc& d, cudaStream_t stream) {
  load_driver_entry_points();
  if (!g_encode_tiled || !g_encode_im2col) return cudaErrorNotSupported;
  if (d.M <= 0 || d.N <= 0) return cudaSuccess;
  if (d.band && !d.bn_out && !d.stats_bwd && !d.replay && !d.stats_acc && d.a_kind == Operand::Im2colK && gemm_band_ok(d) &&
      (d.band == 2 || gemm_band_preferred(d)))
    return gemm_band_launch(d, stream);
  const int bn = gemm_block_n(d);
  if (bn != 64 && bn != 128 && bn != 256) return cudaErrorInvalidValue;
  if (d.stats && d.out_f32) return cudaErrorInvalidValue;  // statistics are of the stored bf16 values
  if (d.stats_bwd && (!d.stats || !d.bs_y || !d.bs_mean || !d.bs_scale || !d.bs_shift || d.splits > 1 || d.remap ||
                      d.accumulate_out || d.bn_out || d.N % 8 || d.bs_ldy % 8 ||
                      (reinterpret_cast<uintptr_t>(d.bs_y) & 15) || (reinterpret_cast<uintptr_t>(d.out) & 15)))
    return cudaErrorInvalidValue;
  if (d.replay && (!d.stats_bwd || d.block_n == 0)) return cudaErrorInvalidValue;

  KParams kp;
  std::memset(&kp, 0, sizeof(kp));
  kp.M = d.M;
  kp.N = d.N;
  kp.K = d.K;
  kp.stats_bwd = d.stats_bwd ? 1 : 0;
  kp.replay = d.replay ? 1 : 0;
  kp.bs_y = static_cast<const __nv_bfloat16*>(d.bs_y);
  kp.bs_ldy = d.bs_ldy;
  kp.bs_mean = d.bs_mean;
  kp.bs_scale = d.bs_scale;
  kp.bs_shift = d.bs_shift;
  if (d.replay) {
    // statistics replay: no operands, no output write; same tile space
    kp.num_kb = 1;
    kp.kb_per_split = 1;
    kp.out = d.out;
    kp.ldc = d.ldc;
    kp.stats = d.stats;
    const int m_tiles = gemm_m_tiles(d), n_tiles = (d.N + bn - 1) / bn;
    switch (bn) {
      case 64: return launch_bn<64>(kp, m_tiles, n_tiles, 1, 0, false, stream);
      case 128: return launch_bn<128>(kp, m_tiles, n_tiles, 1, 0, false, stream);
      default: return launch_bn<256>(kp, m_tiles, n_tiles, 1, 0, false, stream);
    }
  }
  kp.a_kind = (int)d.a_kind;
  kp.b_kind = (int)d.b_kind;
  // CTA pair: M = 256 tiles, each CTA staging half of B (K-major: a box of
  // bn/2 rows; MN-major: whole 64-wide boxes, so bn >= 128)
  const int pmode = d.pair != 0 ? (d.pair > 0 ? 2 : 0) : pair_mode();
  bool pair = pmode > 0 && !d.stats_bwd && gemm_m_tiles(d) >= 2 && (d.b_kind == Operand::KMajor2D || bn >= 128);
  if (pair && pmode == 1) {
    // measured (tools/gemm_probe.py, profiles/gemm_pair_r2.txt): pairs speed
    // up long plain-operand main loops (+11 % at K = 4608, 8192^3 1.28 ->
    // 1.42 PFLOP/s) but slow epilogue-bound launches (K = 64: -50 %) and
    // gain nothing when A comes through TMA im2col (the load feed bounds it)
    const int splits_ = d.splits < 1 ? 1 : d.splits;
    const long kb_tile = ((d.a_kind == Operand::Im2colK ? (long)d.a_geom.R * d.a_geom.S * ((d.a_geom.C + 63) / 64)
                                                        : (long)(d.K + 63) / 64) +
                          splits_ - 1) / splits_;
    pair = d.a_kind != Operand::Im2colK && kb_tile >= 32;
  }
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
                     64, pair ? bn / 2 : bn);
      break;
    case Operand::MNMajor2D:
      ok = encode_2d(&kp.tb, d.b, d.b_extent > 0 ? d.b_extent : d.N, d.K, d.b_ld, 64, 64);
      break;
    case Operand::Im2colMN:
      geo = &d.b_geom;
      ok = encode_im2col(&kp.tb, d.b, d.b_geom, 64);
      break;
    case Operand::WeightTapsMN: {
      // [Cout][taps][Cpad] viewed as {ci (valid extent), tap, co}; a box is a
      // 64 (ci) x 64 (co) tile of one tap: MN-major with K = co rows
      cuuint64_t dims[3] = {(cuuint64_t)(d.b_extent > 0 ? d.b_extent : d.N), (cuuint64_t)d.b_taps,
                            (cuuint64_t)d.b_rows};
      cuuint64_t strides[2] = {(cuuint64_t)d.b_cpad * 2, (cuuint64_t)d.b_taps * d.b_cpad * 2};
      cuuint32_t box[3] = {64, 1, 64};
      cuuint32_t es[3] = {1, 1, 1};
      ok = g_encode_tiled(&kp.tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(d.b), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      kp.b_taps = d.b_taps;
      if (d.b_tap_base >= 0) {
        kp.b_tap_base = d.b_tap_base, kp.b_tap_dr = d.b_tap_dr, kp.b_tap_ds = d.b_tap_ds;
      } else {
        kp.b_tap_base = d.b_taps - 1, kp.b_tap_dr = d.a_geom.S, kp.b_tap_ds = 1;
      }
      if (d.a_kind != Operand::Im2colK) return cudaErrorInvalidValue;  // 1x1 dgrad uses MNMajor2D
      break;
    }
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
  kp.stats_acc = d.stats_acc ? 1 : 0;
  kp.split_stride = d.split_stride;
  // output through TMA (store, or reduce-add when accumulating) whenever the
  // rows are not remapped and the strides are 16-byte multiples
  {
    const int es = d.out_f32 ? 4 : 2;
    const long sstride = splits > 1 ? d.split_stride : (long)d.M * d.ldc;
    if (!d.remap && d.out && ((long)d.ldc * es) % 16 == 0 && (sstride * es) % 16 == 0 &&
        (reinterpret_cast<uintptr_t>(d.out) & 15) == 0) {
      cuuint64_t dims[3] = {(cuuint64_t)d.N, (cuuint64_t)d.M, (cuuint64_t)splits};
      cuuint64_t strides[2] = {(cuuint64_t)d.ldc * es, (cuuint64_t)sstride * es};
      cuuint32_t box[3] = {d.out_f32 ? 16u : 32u, 32u, 1u};
      cuuint32_t estr[3] = {1, 1, 1};
      if (g_encode_tiled(&kp.tc, d.out_f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                         d.out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
        kp.out_mode = d.accumulate_out ? 2 : 1;
    }
  }
  if (d.bn_out) {
    // fused BN apply: needs the TMA-store epilogue, a plain bf16 output and
    // 16-byte aligned per-channel parameters
    if (kp.out_mode != 1 || d.out_f32 || splits > 1 || d.stats || d.N % 8 ||
        (reinterpret_cast<uintptr_t>(d.bn_out) & 15) || (reinterpret_cast<uintptr_t>(d.bn_scale) & 15) ||
        (reinterpret_cast<uintptr_t>(d.bn_shift) & 15))
      return cudaErrorInvalidValue;
    cuuint64_t dims[3] = {(cuuint64_t)d.N, (cuuint64_t)d.M, 1};
    cuuint64_t strides[2] = {(cuuint64_t)d.ldc * 2, (cuuint64_t)d.M * d.ldc * 2};
    cuuint32_t box[3] = {32u, 32u, 1u};
    cuuint32_t estr[3] = {1, 1, 1};
    if (g_encode_tiled(&kp.tc2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d.bn_out, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    kp.fuse_bn = 1;
    kp.bn_scale = d.bn_scale;
    kp.bn_shift = d.bn_shift;
    kp.bn_relu = d.bn_relu ? 1 : 0;
  }
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
    case 64: return launch_bn<64>(kp, m_tiles, n_tiles, splits, d.max_ctas, pair, stream);
    case 128: return launch_bn<128>(kp, m_tiles, n_tiles, splits, d.max_ctas, pair, stream);
    default: return launch_bn<256>(kp, m_tiles, n_tiles, splits, d.max_ctas, pair, stream);
  }
}

}  // namespace rfk
