// Micro-benchmark of tcgen05.mma issue cost (timing only, results unused):
// one CTA per SM issues back-to-back 128 x N x 16 bf16 MMAs and reports
// cycles per instruction for
//   SS: A and B from shared memory (the GEMM engine's mode)
//   TS: A from TMEM, B from shared memory
// with a commit every `per_commit` MMAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1808_00079_b200/csrc \
//        tools/mma_micro.cu -o gpurun_out/mma_micro -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "kernels/ptx.cuh"

using namespace rfk;

__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_bench(int iters, int per_commit, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bars[1025];
  __shared__ uint32_t tslot;
  // 64 KB of operand space, zeros
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  for (int i = threadIdx.x; i < 1025; i += blockDim.x) mbar_init(&bars[i], 1);
  fence_barrier_init();
  if (threadIdx.x < 32) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x < 32) {
    const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 16384);
    long long t0 = 0, t1 = 0;
    const int commits = (iters - 1) / per_commit + 1;
    for (int rep = 0; rep < 2; ++rep) {
      __syncwarp();
      t0 = clock64();
      if (elect_one()) {
        // descriptors hoisted: the loop body is the MMAs (+ one commit per 4)
        uint64_t da[4], db[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          da[kk] = umma_desc_sw128(sa + kk * 32, 16, 1024);
          db[kk] = umma_desc_sw128(sb + kk * 32, 16, 1024);
        }
        for (int i = 0; i < iters; i += 4) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if (TS)
              umma_ts(tmem, tmem + 256 + kk * 8, db[kk], idesc, 1u);
            else
              umma_bf16(tmem, da[kk], db[kk], idesc, 1u);
          }
          if (per_commit == 4 && i + 4 < iters) umma_commit(&bars[i >> 2]);
        }
        umma_commit(&bars[commits - 1]);
      }
      __syncwarp();
      // every barrier gets one arrival per rep; the commits complete in order
      mbar_wait(&bars[commits - 1], rep & 1);
      t1 = clock64();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, bool TS>
void run(int iters, int per_commit, long long* d) {
  auto k = mma_bench<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k<<<148, 128, 70000>>>(iters, per_commit, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0, sum = 0;
  for (int i = 0; i < 148; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    sum += h[i];
  }
  printf("%s N=%3d iters %5d commit/%d: %.1f cycles/MMA (mean), %.1f (max); floor %d\n", TS ? "TS" : "SS", N, iters,
         per_commit, (double)sum / 148 / iters, (double)mx / iters, 128 * N / 256);
}


__device__ __forceinline__ void wait_raw(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Producer / consumer ring handshake (the GEMM's full / empty barriers):
// warp 0 waits empty[s] and arrives on full[s]; warp 1 waits full[s], issues
// `mmas` MMAs (128 x 256 x 16) and releases the stage with tcgen05.commit
// (mode 0) or a plain mbarrier arrive (mode 1).
template <int V>
__global__ void __launch_bounds__(128, 1) ring_bench(int iters, int depth, int mode, int mmas, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[16], empty[16];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x < 16) {
    mbar_init(&full[threadIdx.x], 1);
    mbar_init(&empty[threadIdx.x], 1);
  }
  fence_barrier_init();
  if (threadIdx.x >= 32 && threadIdx.x < 64) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  const long long t0 = clock64();
  if (threadIdx.x < 32) {
    int s = 0;
    uint32_t ph = 0;
    if (V == 0) {
      for (int i = 0; i < iters; ++i) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) mbar_arrive(&full[s]);
        __syncwarp();
        if (++s == depth) s = 0, ph ^= 1;
      }
    } else if (threadIdx.x == 0) {  // one thread, raw wait
      for (int i = 0; i < iters; ++i) {
        wait_raw(&empty[s], ph ^ 1);
        mbar_arrive(&full[s]);
        if (++s == depth) s = 0, ph ^= 1;
      }
    }
  } else if (threadIdx.x < 64) {
    const uint32_t idesc = umma_idesc_bf16(128, 256, false, false);
    const uint64_t da = umma_desc_sw128(smem_u32(smem), 16, 1024), db = umma_desc_sw128(smem_u32(smem + 16384), 16, 1024);
    int s = 0;
    uint32_t ph = 0;
    if (V == 0) {
      for (int i = 0; i < iters; ++i) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          for (int k = 0; k < mmas; ++k) umma_bf16(tmem, da, db, idesc, 1u);
          if (mode == 0) umma_commit(&empty[s]);
          else mbar_arrive(&empty[s]);
        }
        __syncwarp();
        if (++s == depth) s = 0, ph ^= 1;
      }
    } else if (threadIdx.x == 32) {
      for (int i = 0; i < iters; ++i) {
        wait_raw(&full[s], ph);
        tc_fence_after();
        for (int k = 0; k < mmas; ++k) umma_bf16(tmem, da, db, idesc, 1u);
        if (mode == 0) umma_commit(&empty[s]);
        else mbar_arrive(&empty[s]);
        if (++s == depth) s = 0, ph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (threadIdx.x >= 32 && threadIdx.x < 64) tmem_dealloc<512>(tmem);
}

template <int V>
void ring(int iters, int depth, int mode, int mmas, long long* d) {
  cudaFuncSetAttribute(ring_bench<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  ring_bench<V><<<148, 128, 70000>>>(iters, depth, mode, mmas, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return;
  }
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long sum = 0;
  for (int i = 0; i < 148; ++i) sum += h[i];
  printf("V%d ring depth %2d %s, %d MMAs (N=256) per stage: %.1f cycles per stage\n", V, depth,
         mode == 0 ? "tcgen05.commit" : "mbarrier.arrive", mmas, (double)sum / 148 / iters);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int pc : {4}) {
    run<64, false>(4096, pc, d);
    run<128, false>(4096, pc, d);
    run<256, false>(4096, pc, d);
    run<64, true>(4096, pc, d);
    run<128, true>(4096, pc, d);
    run<256, true>(4096, pc, d);
  }
  for (int depth : {4, 8})
    for (int mode : {0, 1})
      for (int mmas : {0, 1, 4}) {
        if (mode == 1 && mmas > 0) continue;
        ring<0>(20000, depth, mode, mmas, d);
        ring<1>(20000, depth, mode, mmas, d);
      }
  return 0;
}
