// Shifted-band implicit GEMM for stride-1 R x S convolutions on sm_100a.
//
// The TMA im2col mode re-fetches every input pixel once per filter tap and
// runs at about a third of the tiled-mode rate, which made the 3x3 convs of
// ResNet / DenseNet A-load bound (~0.5 us per 128-pixel K block whatever the
// tile width).  Here the output is indexed in "plane" coordinates: image n,
// output row h, padded column w' (0 <= w' < Wp = W + 2 pad_w; columns w' >= Q
// are junk).  Output position j = h * Wp + w' reads padded input position
// j + r * Wp + s for tap (r, s), so for one 64-channel chunk the A operands
// of all R * S taps are 128-row windows of ONE band of padded input rows.
// The band is a single tiled 4-D TMA box {64 ch, Wp, BR rows, 1 image} whose
// out-of-bounds columns / rows are zero-filled (= the convolution padding);
// each tap's MMA reads it through a descriptor whose start row is shifted by
// r * Wp + s (the swizzle is a function of the absolute smem address, so any
// 128-byte row of the band is a valid operand start).
// A traffic drops ~R*S / (1 + halo) fold and the loads are tiled-mode.
//
//   warp 0      TMA producer: band ring (2 deep) + weight ring
//   warp 1      TMEM allocator + MMA issuer
//   warps 2..9  epilogue: TMEM -> regs -> [stats] -> plane -> NHWC row map
//
// Used for conv fprop (B = K-major weights) and for the stride-1 form of conv
// dgrad (B = the flipped weight taps read in place).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "kernels/kernels.h"
#include "kernels/launch.cuh"
#include "kernels/ptx.cuh"

#ifndef RFK_GEMM_TUNING
#define RFK_GEMM_TUNING 0
#endif

namespace rfk {

namespace {

constexpr int kBM = 128;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps + 32;  // + the band fix-up warp (flat mode)
constexpr int kSmemMax = 232448;
constexpr int kStaging = kEpiWarps * 2048;

struct alignas(64) BandParams {
  CUtensorMap ta;  // 4-D tiled map over the NHWC input {C, W, H, N}, box {64, Wp, BR, 1}
  CUtensorMap tb;  // weights
  CUtensorMap ta2;  // flat mode: the input as a 2-D [N*H*W pixels][C] map, box {64, Wp}
  int N;                       // GEMM N (output channels)
  int cblocks, taps, R, S;     // K = taps x cblocks x 64
  int Wp, P, Q, ph, pw, BR;    // plane geometry
  int plane;                   // P * Wp positions per image
  int tiles_per_img, m_tiles, n_tiles;
  int tile_pos;                // plane positions per tile: whole output rows (rows x Wp <= 128), else 128
  int b_kind;                  // 0 K-major weights (fprop), 4 flipped weight taps (dgrad)
  void* out;
  long ldc;
  int accumulate_out;
  float* stats;
  int band_bytes;              // smem bytes of one band stage (1024-aligned)
  int box_bytes;               // bytes the band TMA delivers
  int b_stages;
  int band_stages;  // band ring depth (2..4)
  int row_boxes;   // band as BR one-row boxes instead of one BR-row box (tuning)
  int prefetch_tiles;  // L2 prefetch distance in tiles of this CTA (0 = off)
  int flat;        // band rows as 2-D boxes over the flat pixel array + fix-up of the padding lines
  int H, W;
  int b_resident;  // all taps x chunks of B fit the ring: loaded once per CTA, never released
  int experiment;  // tuning only: 2 drop the output, 4 also skip the MMAs
  unsigned long long* dbg;  // tuning only: per-tile timestamps of CTA 0
};

__device__ __forceinline__ uint64_t desc_sw128_rows(uint32_t addr) {
  // K-major SW128: LBO unused (16), SBO = 8 rows x 128 B.  The start row may
  // be any row of the band: the hardware applies the 128-byte swizzle on the
  // absolute shared-memory address (as the TMA wrote it), so the descriptor's
  // base-offset field stays 0 (measured: a row-phase base offset corrupts
  // every shifted tap, zero is exact).
  return umma_desc_sw128(addr, 16, 1024);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) gemm_band_kernel(const __grid_constant__ BandParams p) {
  constexpr int kTileB = BN * 64 * 2;
  constexpr int kTmemCols = BN;
  constexpr int HB = BN / 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* band = smem;                                       // [band_stages][band_bytes]
  uint8_t* bring = band + p.band_stages * p.band_bytes;       // [b_stages][kTileB]
  uint8_t* stage_buf = bring + p.b_stages * kTileB;  // epilogue staging, then column sums
  float* wsum = reinterpret_cast<float*>(stage_buf + kStaging);
  uint64_t* band_full = reinterpret_cast<uint64_t*>(wsum + kEpiWarps * 2 * HB);
  uint64_t* band_empty = band_full + 4;
  uint64_t* band_ready = band_empty + 4;  // flat mode: padding lines zeroed
  uint64_t* b_full = band_ready + 4;
  uint64_t* b_empty = b_full + p.b_stages;
  uint64_t* acc_full = b_empty + p.b_stages;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t warp = warp_id();
  const int total = p.m_tiles * p.n_tiles;

  if (warp == 0 && elect_one()) {
    tma_prefetch(p.flat ? &p.ta2 : &p.ta);
    tma_prefetch(&p.tb);
    for (int s = 0; s < p.band_stages; ++s) {
      mbar_init(&band_full[s], 1);
      mbar_init(&band_empty[s], 1);
      mbar_init(&band_ready[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], kEpiWarps);
    }
    for (int s = 0; s < p.b_stages; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<2 * kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_enter();

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (elect_one()) {
      int bs = 0, s = 0;
      uint32_t bph = 0, ph = 0;
      if (p.b_resident) {  // single n tile: every weight tile once, kept for all M tiles
        for (int cb = 0; cb < p.cblocks; ++cb)
          for (int tap = 0; tap < p.taps; ++tap) {
            const int slot = cb * p.taps + tap;
            uint8_t* sb = bring + slot * kTileB;
            mbar_arrive_expect_tx(&b_full[slot], kTileB);
            if (p.b_kind == 0) {
              tma_load_2d(sb, &p.tb, &b_full[slot], (tap * p.cblocks + cb) * 64, 0);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_3d(sb + j * 8192, &p.tb, &b_full[slot], 64 * j, p.taps - 1 - tap, cb * 64);
            }
          }
      }
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int mt = t % p.m_tiles, n0 = (t / p.m_tiles) * BN;
        const int img = mt / p.tiles_per_img, j0 = (mt % p.tiles_per_img) * p.tile_pos;
        const int rho0 = j0 / p.Wp;
        // warm L2 with this CTA's band a few tiles ahead: the band loads are
        // DRAM-latency bound with only band_stages of them in shared memory
        if (p.prefetch_tiles > 0) {
          const int tf = t + p.prefetch_tiles * (int)gridDim.x;
          if (tf < total) {
            const int mf = tf % p.m_tiles;
            const int imf = mf / p.tiles_per_img, jf = (mf % p.tiles_per_img) * p.tile_pos;
            for (int cbf = 0; cbf < p.cblocks; ++cbf)
              tma_prefetch_l2_4d(&p.ta, cbf * 64, -p.pw, jf / p.Wp - p.ph, imf);
          }
        }
        for (int cb = 0; cb < p.cblocks; ++cb) {
          mbar_wait(&band_empty[bs], bph ^ 1);
          if (p.dbg && blockIdx.x == 0 && t / gridDim.x < 16) p.dbg[(t / gridDim.x) * 4 + 0] = global_ns();
          if (p.flat) {
            // one 2-D box of Wp consecutive pixels per band row that lies in
            // the image; the fix-up warp zeroes the rest
            int valid = 0;
            for (int rr = 0; rr < p.BR; ++rr) {
              const int h = rho0 - p.ph + rr;
              valid += (h >= 0 && h < p.H) ? 1 : 0;
            }
            mbar_arrive_expect_tx(&band_full[bs], (uint32_t)(valid * p.Wp * 128));
            for (int rr = 0; rr < p.BR; ++rr) {
              const int h = rho0 - p.ph + rr;
              if (h < 0 || h >= p.H) continue;
              tma_load_2d(band + bs * p.band_bytes + rr * p.Wp * 128, &p.ta2, &band_full[bs], cb * 64,
                          (img * p.H + h) * p.W - p.pw);
            }
          } else
          mbar_arrive_expect_tx(&band_full[bs], p.box_bytes);
          if (p.flat) {
          } else if (p.row_boxes) {  // one {64, Wp, 1, 1} box per band row
            for (int rr = 0; rr < p.BR; ++rr)
              tma_load_4d(band + bs * p.band_bytes + rr * p.Wp * 128, &p.ta, &band_full[bs], cb * 64, -p.pw,
                          rho0 - p.ph + rr, img);
          } else {
            tma_load_4d(band + bs * p.band_bytes, &p.ta, &band_full[bs], cb * 64, -p.pw, rho0 - p.ph, img);
          }
          if (++bs == p.band_stages) {
            bs = 0;
            bph ^= 1;
          }
          for (int tap = 0; tap < p.taps && !p.b_resident; ++tap) {
            mbar_wait(&b_empty[s], ph ^ 1);
            uint8_t* sb = bring + s * kTileB;
            mbar_arrive_expect_tx(&b_full[s], kTileB);
            if (p.b_kind == 0) {
              tma_load_2d(sb, &p.tb, &b_full[s], (tap * p.cblocks + cb) * 64, n0);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_3d(sb + j * 8192, &p.tb, &b_full[s], n0 + 64 * j, p.taps - 1 - tap, cb * 64);
            }
            if (++s == p.b_stages) {
              s = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const bool b_mn = p.b_kind != 0;
    const uint32_t idesc = umma_idesc_bf16(kBM, BN, false, b_mn);
    int bs = 0, s = 0, local = 0;
    uint32_t bph = 0, ph = 0;
    // resident weights: every slot is loaded once, wait for all of them up front
    // (a wait on a completed barrier still costs ~90 cycles + the fence; per
    // tap that bounded the issue loop)
    if (p.b_resident && (int)blockIdx.x < total) {
      for (int slot = 0; slot < p.cblocks * p.taps; ++slot) mbar_wait(&b_full[slot], 0u);
      tc_fence_after();
    }
    const uint32_t bhi = (uint32_t)((b_mn ? umma_desc_sw128(0, 8192, 1024) : umma_desc_sw128(0, 16, 1024)) >> 32);
    const uint32_t blo_k = (uint32_t)(b_mn ? umma_desc_sw128(0, 8192, 1024) : umma_desc_sw128(0, 16, 1024));
    const uint32_t ahi = (uint32_t)(desc_sw128_rows(0) >> 32), alo_k = (uint32_t)desc_sw128_rows(0);
    const uint32_t b_kstep = b_mn ? (2048u >> 4) : (32u >> 4);
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int mt = t % p.m_tiles;
      const int j0 = (mt % p.tiles_per_img) * p.tile_pos;
      const int row0 = j0 - (j0 / p.Wp) * p.Wp;  // first output row's offset inside the band
      const int acc = local & 1;
      mbar_wait(&acc_empty[acc], ((local >> 1) & 1) ^ 1);
      tc_fence_after();
      if (p.dbg && blockIdx.x == 0 && local < 16 && lane_id() == 0) p.dbg[local * 4 + 3] = global_ns();
      const uint32_t d_tmem = tmem + (uint32_t)(acc * kTmemCols);
      for (int cb = 0; cb < p.cblocks; ++cb) {
        mbar_wait(p.flat ? &band_ready[bs] : &band_full[bs], bph);
        tc_fence_after();
        if (p.dbg && blockIdx.x == 0 && local < 16 && cb == 0 && lane_id() == 0) p.dbg[local * 4 + 1] = global_ns();
        const uint32_t sa0 = smem_u32(band + bs * p.band_bytes);
        if (p.b_resident) {
          // all taps of this channel block in one tight issue loop: the A
          // start row advances by one per filter column and by Wp per row
          if (elect_one()) {
            const uint32_t a_base = alo_k + ((sa0 + (uint32_t)row0 * 128u) >> 4);
            const uint32_t b_base = blo_k + (smem_u32(bring + cb * p.taps * kTileB) >> 4);
            int r = 0, c = 0;
            for (int tap = 0; tap < p.taps; ++tap) {
              const uint32_t a_lo = a_base + (uint32_t)(r * p.Wp + c) * 8u;  // 128-byte rows, >> 4
              const uint32_t b_lo = b_base + (uint32_t)tap * (uint32_t)(kTileB >> 4);
#pragma unroll
              for (int kk = 0; kk < ((RFK_GEMM_TUNING && p.experiment == 4) ? 0 : 4); ++kk) {
                const uint64_t da = ((uint64_t)ahi << 32) | (a_lo + (uint32_t)kk * 2u);
                const uint64_t db = ((uint64_t)bhi << 32) | (b_lo + (uint32_t)kk * b_kstep);
                umma_bf16(d_tmem, da, db, idesc, (cb > 0 || tap > 0 || kk > 0) ? 1u : 0u);
              }
              if (++c == p.S) {
                c = 0;
                ++r;
              }
            }
            umma_commit(&band_empty[bs]);
            if (cb + 1 == p.cblocks) umma_commit(&acc_full[acc]);
          }
          __syncwarp();
        }
        for (int tap = 0; tap < p.taps && !p.b_resident; ++tap) {
          const int slot = p.b_resident ? cb * p.taps + tap : s;
          mbar_wait(&b_full[slot], p.b_resident ? 0u : ph);
          tc_fence_after();
          if (elect_one()) {
            const int r = tap / p.S, c = tap - r * p.S;
            const uint32_t row = (uint32_t)(row0 + r * p.Wp + c);
            const uint32_t sa = sa0 + row * 128u;
            const uint32_t sb = smem_u32(bring + slot * kTileB);
#pragma unroll
            for (int kk = 0; kk < ((RFK_GEMM_TUNING && p.experiment == 4) ? 0 : 4); ++kk) {
              const uint64_t da = desc_sw128_rows(sa + kk * 32);
              const uint64_t db = b_mn ? umma_desc_sw128(sb + kk * 2048, 8192, 1024) : umma_desc_sw128(sb + kk * 32, 16, 1024);
              umma_bf16(d_tmem, da, db, idesc, (cb > 0 || tap > 0 || kk > 0) ? 1u : 0u);
            }
            if (!p.b_resident) umma_commit(&b_empty[s]);
            if (tap + 1 == p.taps) {
              umma_commit(&band_empty[bs]);
              if (cb + 1 == p.cblocks) umma_commit(&acc_full[acc]);
            }
          }
          __syncwarp();
          if (!p.b_resident && ++s == p.b_stages) {
            s = 0;
            ph ^= 1;
          }
        }
        if (++bs == p.band_stages) {
          bs = 0;
          bph ^= 1;
        }
      }
    }
  } else if (warp == 2 + kEpiWarps) {
    // ------------------------------------------------ band fix-up (flat mode)
    // Zero the band lines the flat 2-D boxes filled with neighbouring pixels
    // (columns outside the image) or never loaded (rows outside the image),
    // then publish the band to the MMA warp.
    if (p.flat) {
      const uint32_t lane = lane_id();
      int bs = 0;
      uint32_t bph = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int mt = t % p.m_tiles;
        const int j0 = (mt % p.tiles_per_img) * p.tile_pos;
        const int rho0 = j0 / p.Wp;
        for (int cb = 0; cb < p.cblocks; ++cb) {
          mbar_wait(&band_full[bs], bph);
          uint8_t* b0 = band + bs * p.band_bytes;
          for (int rr = 0; rr < p.BR; ++rr) {
            const int h = rho0 - p.ph + rr;
            const bool row_in = h >= 0 && h < p.H;
            // lines of this row to clear: all of them, or the pad columns
            const int n_lines = row_in ? (p.Wp - p.W) : p.Wp;
            for (int i = (int)lane; i < n_lines * 8; i += 32) {
              const int li = i >> 3, chunk = i & 7;
              int col;
              if (!row_in) col = li;
              else col = li < p.pw ? li : p.W + li;  // [0, pw) and [pw + W, Wp)
              *reinterpret_cast<uint4*>(b0 + (rr * p.Wp + col) * 128 + chunk * 16) = make_uint4(0u, 0u, 0u, 0u);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&band_ready[bs]);
          if (++bs == p.band_stages) {
            bs = 0;
            bph ^= 1;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------ epilogue (warps 2..9)
    // Plane rows -> NHWC pixel rows (junk columns w' >= Q and positions past
    // the image's plane are dropped and contribute zeros to the statistics),
    // bf16 staging, 64-byte row segments (4 lanes per row), optional
    // accumulate, fused BN column sums of the stored bf16 values.
    const uint32_t quarter = warp & 3, half = (warp - 2) >> 2, ew = warp - 2, lane = lane_id();
    uint8_t* gb = stage_buf + ew * 2048;
    float* my_sum = wsum + ew * 2 * HB;
    int cur_nt = -1;
    auto flush_stats = [&](int nt) {
      asm volatile("bar.sync 1, 256;" ::: "memory");
      float* rowp = p.stats + (long)blockIdx.x * 2 * p.N;
      for (int c = (int)(ew * 32 + lane); c < BN; c += 256) {
        const int j = c >> 5, h = j & 1, lc = ((j >> 1) << 5) + (c & 31);
        float s0 = 0.f, q0 = 0.f;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const float* ws = wsum + (4 * h + ((qq + 2) & 3)) * 2 * HB;
          s0 += ws[lc];
          q0 += ws[HB + lc];
        }
        const int col = nt * BN + c;
        if (col < p.N) {
          rowp[col] = s0;
          rowp[p.N + col] = q0;
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
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int mt = t % p.m_tiles, nt = t / p.m_tiles;
      const int img = mt / p.tiles_per_img, j0 = (mt % p.tiles_per_img) * p.tile_pos;
      const int acc = local & 1;
      if (p.stats && nt != cur_nt) {
        if (cur_nt >= 0) flush_stats(cur_nt);
        cur_nt = nt;
      }
      mbar_wait(&acc_full[acc], (local >> 1) & 1);
      tc_fence_after();
      if (p.dbg && blockIdx.x == 0 && local < 16 && ew == 0 && lane == 0) p.dbg[local * 4 + 2] = global_ns();
      const int jl = j0 + (int)(quarter * 32 + lane);  // this lane's plane position
      const bool row_ok = jl - j0 < p.tile_pos && jl < p.plane && (jl % p.Wp) < p.Q;
#pragma unroll 1
      for (int c0 = (int)half * 32; c0 < BN; c0 += 64) {
        uint32_t r[32];
        tmem_ld32(tmem + (uint32_t)(acc * kTmemCols) + ((quarter * 32u) << 16) + (uint32_t)c0, r);
        tmem_ld_wait();
        if (c0 + 64 >= BN) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[acc]);
        }
        const int col0 = nt * BN + c0;
        if (col0 >= p.N || (RFK_GEMM_TUNING && p.experiment >= 2)) continue;
        const bool full_cols = col0 + 32 <= p.N;
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          w[i] = row_ok ? pack_bf16(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])) : 0u;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t sw = (uint32_t)j ^ ((lane >> 1) & 3u);
          *reinterpret_cast<uint4*>(gb + lane * 64 + sw * 16) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
        }
        __syncwarp();
#pragma unroll 1
        for (int it = 0; it < 4; ++it) {
          const uint32_t rr = it * 8 + (lane >> 2), chunk = lane & 3;
          const int jr = j0 + (int)(quarter * 32 + rr);
          if (jr >= p.plane || jr - j0 >= p.tile_pos) continue;
          const int h = jr / p.Wp, wq = jr - h * p.Wp;
          if (wq >= p.Q || !(full_cols || col0 + (int)chunk * 8 < p.N)) continue;
          const uint4 val = *reinterpret_cast<const uint4*>(gb + rr * 64 + ((chunk ^ ((rr >> 1) & 3u)) * 16));
          const long orow = ((long)img * p.P + h) * p.Q + wq;
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.out) + orow * p.ldc + col0 + chunk * 8;
          if (full_cols || col0 + (int)chunk * 8 + 8 <= p.N) {
            uint4 o = val;
            if (p.accumulate_out) {
              const uint4 prev = *reinterpret_cast<const uint4*>(dst);
              const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&val);
              const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&prev);
              __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 fa = __bfloat1622float2(a2[e]), fb = __bfloat1622float2(b2[e]);
                o2[e] = __floats2bfloat162_rn(fa.x + fb.x, fa.y + fb.y);
              }
            }
            *reinterpret_cast<uint4*>(dst) = o;
          } else {
            const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&val);
            for (int e = 0; e < 8 && col0 + (int)chunk * 8 + e < p.N; ++e)
              dst[e] = p.accumulate_out ? __float2bfloat16_rn(__bfloat162float(dst[e]) + __bfloat162float(vb[e])) : vb[e];
          }
        }
        if (p.stats) {
          const uint32_t cp = lane & 15, par = lane >> 4;
          float s0 = 0.f, s1 = 0.f, q0 = 0.f, q1 = 0.f;
#pragma unroll
          for (int rr = 0; rr < 16; ++rr) {
            const uint32_t row = 2 * rr + par;
            const uint32_t off = row * 64 + (((cp >> 2) ^ ((row >> 1) & 3u)) * 16) + (cp & 3) * 4;
            const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(gb + off));
            s0 += f.x;
            s1 += f.y;
            q0 = fmaf(f.x, f.x, q0);
            q1 = fmaf(f.y, f.y, q1);
          }
          s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
          s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
          q0 += __shfl_xor_sync(0xffffffffu, q0, 16);
          q1 += __shfl_xor_sync(0xffffffffu, q1, 16);
          if (lane < 16) {
            const int lc = ((c0 >> 6) << 5) + 2 * (int)lane;
            my_sum[lc] += s0;
            my_sum[lc + 1] += s1;
            my_sum[HB + lc] += q0;
            my_sum[HB + lc + 1] += q1;
          }
        }
        __syncwarp();
      }
    }
    if (p.stats && cur_nt >= 0) flush_stats(cur_nt);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2 * kTmemCols>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_band_encode = nullptr;
std::once_flag g_band_once;

// Band rows one 128-position tile needs: from the tile's first output row to
// its last output row + R - 1 (the tile may start mid-row).
int band_rows(int Wp, int R) { return (Wp - 1 + kBM - 1) / Wp + 1 + (R - 1) + 1; }

template <int BN>
int fixed_smem() {
  return kStaging + kEpiWarps * 2 * (BN / 2) * 4 + 1024 + 512;
}

template <int BN>
cudaError_t band_launch(BandParams& bp, cudaStream_t st) {
  // weights resident when one n tile's taps x chunks fit next to two bands;
  // then as many band stages (<= 4) as the rest of shared memory holds
  const int avail = kSmemMax - fixed_smem<BN>();
  const int tB = BN * 128;
  const int need_b = bp.taps * bp.cblocks * tB;
  bp.b_resident = (bp.n_tiles == 1 && 2 * bp.band_bytes + need_b <= avail) ? 1 : 0;
  bp.b_stages = bp.b_resident ? bp.taps * bp.cblocks : std::min(12, (avail - 2 * bp.band_bytes) / tB);
  if (bp.b_stages < 3 && !bp.b_resident) return cudaErrorInvalidValue;
  bp.band_stages = std::min(4, (avail - bp.b_stages * tB) / bp.band_bytes);
  if (bp.band_stages < 2) return cudaErrorInvalidValue;
  const int smem = bp.band_stages * bp.band_bytes + bp.b_stages * tB + fixed_smem<BN>();
  static int configured = 0;
  if (configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(gemm_band_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    if (e != cudaSuccess) return e;
    configured = kSmemMax;
  }
  static const int experiment = [] {
    const char* e = std::getenv("RFK_GEMM_EXPERIMENT");  // tuning experiments only
    return e ? std::atoi(e) : 0;
  }();
  bp.experiment = experiment;
  static unsigned long long* dbg = nullptr;
  if (std::getenv("RFK_BAND_DEBUG")) {
    if (!dbg) cudaMalloc(&dbg, 64 * 8);
    bp.dbg = dbg;
  }
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int grid = std::min(bp.m_tiles * bp.n_tiles, sms);
  cudaError_t e = launch_k(gemm_band_kernel<BN>, grid, kThreads, smem, st, bp);
  if (bp.dbg && e == cudaSuccess) {  // tuning only: timeline of CTA 0
    unsigned long long h[64];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, bp.dbg, sizeof(h), cudaMemcpyDeviceToHost);
    for (int i = 0; i < 8; ++i)
      printf("tile %d: band issue %+8.0f  band ready %+8.0f  mma start %+8.0f  epi ready %+8.0f ns\n", i,
             (double)(h[i * 4 + 0] - h[0]), (double)(h[i * 4 + 1] - h[0]), (double)(h[i * 4 + 3] - h[0]),
             (double)(h[i * 4 + 2] - h[0]));
  }
  return e;
}

}  // namespace

// Where the band kernel measured faster than TMA im2col (tools/band_probe.py,
// late round 2): 3x3 stride-1 convs at >= 48 output columns (ResNet layer 1,
// DenseNet block 1: 56x56x64 fprop 19.9 -> 17.5 us, dgrad 19.9 -> 15.5 us,
// 56x56x128 -> 32 fprop 34.4 -> 24.8 us) and narrow (<= 32 channel) outputs
// from 24 columns on (28x28x128 -> 32: 12.6 -> 11.5 us).  At 28x28x128 -> 128
// it is slower (20.2 vs 15.1 us), at 14x14 equal.
bool gemm_band_preferred(const GemmDesc& d) {
  const ConvGeom& g = d.a_geom;
  if (g.R != 3 || g.S != 3) return false;
  return g.Q >= 48 || (d.N <= 32 && g.Q >= 24);
}

bool gemm_band_ok(const GemmDesc& d) {
  const ConvGeom& g = d.a_geom;
  if (g.stride_h != 1 || g.stride_w != 1 || g.R * g.S < 2) return false;
  const int Wp = g.W + 2 * g.pad_w;
  if (Wp > 256 || g.Q < 24) return false;  // junk columns (S - 1 of Wp) must stay a small fraction
  const int BR = band_rows(Wp, g.R);
  const int band_bytes = (BR * Wp * 128 + 1023) / 1024 * 1024;
  if (BR > 256 || 2 * band_bytes > 120 * 1024) return false;
  return d.out != nullptr && !d.out_f32 && d.splits <= 1 && !d.remap && !d.bias;
}

cudaError_t gemm_band_launch(const GemmDesc& d, cudaStream_t stream) {
  std::call_once(g_band_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_band_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_band_encode) return cudaErrorNotSupported;
  if (!gemm_band_ok(d)) return cudaErrorInvalidValue;
  const ConvGeom& g = d.a_geom;
  BandParams bp;
  std::memset(&bp, 0, sizeof(bp));
  bp.N = d.N;
  bp.R = g.R;
  bp.S = g.S;
  bp.taps = g.R * g.S;
  bp.cblocks = (g.C + 63) / 64;
  bp.Wp = g.W + 2 * g.pad_w;  // (rounding it up to 8 pixels measured slower)
  bp.P = g.P;
  bp.Q = g.Q;
  bp.ph = g.pad_h;
  bp.pw = g.pad_w;
  bp.plane = g.P * bp.Wp;
  // Row-aligned tiles: a tile is the largest whole number of output rows that
  // fits 128 positions, so its band is exactly rows + R - 1 input rows (at
  // 56x56: 2 rows = 116 positions, a 4-row band instead of the 7 rows a tile
  // starting mid-row needs).  The MMA still reads 128 rows of A; rows past the
  // tile are junk (beyond the band: the next shared-memory region) and the
  // epilogue drops them.  RFK_BAND_ALIGN=0: 128-position tiles; 2: aligned
  // whatever the channel count.
  static const int align = [] {
    const char* e = std::getenv("RFK_BAND_ALIGN");
    return e ? std::atoi(e) : 1;
  }();
  // (measured: aligned wins with two or more 64-channel blocks, whose bands
  // repeat per block -- 56x56x128 -> 32: 43.6 -> 24.8 us -- and loses ~10 %
  // with one, whose 7-row band already fits next to the resident weights)
  const int rpt = bp.Wp <= kBM ? kBM / bp.Wp : 0;
  if (align && rpt >= 1 && (bp.cblocks >= 2 || align == 2)) {
    bp.tile_pos = rpt * bp.Wp;
    bp.BR = std::min(rpt, g.P) + g.R - 1;
    bp.tiles_per_img = (g.P + rpt - 1) / rpt;
  } else {
    bp.tile_pos = kBM;
    bp.BR = band_rows(bp.Wp, g.R);
    bp.tiles_per_img = (bp.plane + kBM - 1) / kBM;
  }
  bp.m_tiles = g.N * bp.tiles_per_img;
  bp.box_bytes = 64 * 2 * bp.Wp * bp.BR;
  bp.band_bytes = (bp.box_bytes + 1023) / 1024 * 1024;
  bp.out = d.out;
  bp.ldc = d.ldc;
  bp.accumulate_out = d.accumulate_out;
  bp.stats = d.stats;
  // band map: NHWC input, box {64 channels, Wp columns, BR rows, 1 image}
  {
    cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    cuuint64_t strides[3] = {(cuuint64_t)g.C * 2, (cuuint64_t)g.W * g.C * 2, (cuuint64_t)g.H * g.W * g.C * 2};
    static const int flat = [] {
      const char* e = std::getenv("RFK_BAND_FLAT");  // tuning experiments only
      return e ? std::atoi(e) : 0;
    }();
    bp.flat = flat;
    static const int pf = [] {
      const char* e = std::getenv("RFK_BAND_PREFETCH");  // tuning experiments only (measured: no gain)
      return e ? std::atoi(e) : 0;
    }();
    bp.prefetch_tiles = pf;
    bp.H = g.H;
    bp.W = g.W;
    {
      cuuint64_t d2[2] = {(cuuint64_t)g.C, (cuuint64_t)g.N * g.H * g.W};
      cuuint64_t s2[1] = {(cuuint64_t)g.C * 2};
      cuuint32_t b2[2] = {64, (cuuint32_t)bp.Wp};
      cuuint32_t e2[2] = {1, 1};
      if (g_band_encode(&bp.ta2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d.a), d2, s2, b2, e2,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    static const int row_boxes = [] {
      const char* e = std::getenv("RFK_BAND_ROWBOX");  // tuning experiments only
      return e ? std::atoi(e) : 0;
    }();
    bp.row_boxes = row_boxes;
    cuuint32_t box[4] = {64, (cuuint32_t)bp.Wp, row_boxes ? 1u : (cuuint32_t)bp.BR, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (g_band_encode(&bp.ta, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(d.a), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  int bn = d.N <= 64 ? 64 : 128;
  if (d.block_n == 64 || d.block_n == 128) bn = d.block_n;
  if (d.b_kind == Operand::KMajor2D) {
    bp.b_kind = 0;
    cuuint64_t dims[2] = {(cuuint64_t)bp.taps * bp.cblocks * 64, (cuuint64_t)d.N};
    cuuint64_t strides[1] = {(cuuint64_t)d.b_ld * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)bn};
    cuuint32_t es[2] = {1, 1};
    if (g_band_encode(&bp.tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(d.b), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else if (d.b_kind == Operand::WeightTapsMN) {
    bp.b_kind = 4;
    cuuint64_t dims[3] = {(cuuint64_t)(d.b_extent > 0 ? d.b_extent : d.N), (cuuint64_t)d.b_taps,
                          (cuuint64_t)d.b_rows};
    cuuint64_t strides[2] = {(cuuint64_t)d.b_cpad * 2, (cuuint64_t)d.b_taps * d.b_cpad * 2};
    cuuint32_t box[3] = {64, 1, 64};
    cuuint32_t es[3] = {1, 1, 1};
    if (g_band_encode(&bp.tb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(d.b), dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  } else {
    return cudaErrorInvalidValue;
  }
  bp.n_tiles = (d.N + bn - 1) / bn;
  return bn == 64 ? band_launch<64>(bp, stream) : band_launch<128>(bp, stream);
}

}  // namespace rfk
