// MMA-issuer loop microbenchmark (tuning tool, not part of the product): the
// per-K-block work of the executor's MMA warp -- wait for a ring stage, issue
// 4 tcgen05.mma (M = 128, K = 16 each) from that stage, commit the stage back --
// with the stage barriers signalled by this thread's own commits `lag` K blocks
// earlier (operands resident; no producer), in three code shapes:
//   mode 0: the whole warp walks the loop, elect.sync + __syncwarp per K block,
//           descriptors rebuilt from the stage address (the executor today);
//   mode 1: one thread walks the loop, descriptors rebuilt per K block;
//   mode 2: one thread, descriptors advanced by a per-stage constant (adds only);
//   mode 3: whole warp, stages of 2 K blocks: one wait + 8 MMAs + one commit;
//   mode 4: as mode 3 with a wait and a commit per K block;
//   mode 5: one wait, two commits per 2-K-block stage; mode 6: two waits, two commits,
//           the second wait on the first commit's barrier (modes 3-6: N <= 128).
// nofence = 1 drops the tcgen05.fence::after_thread_sync after each stage wait.
// Reports SM cycles per K block and the fraction of the tensor floor (4 x 128 N / 256).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2109_01611_b200/csrc \
//        tools/mma_loop_micro.cu -o tools/mma_loop_micro && ./tools/mma_loop_micro
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

constexpr uint32_t kStage = 48 * 1024;

__global__ void __launch_bounds__(128, 1) mma_loop(int n, int kb, int lag, int mode, int nofence, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(base + 4 * kStage);
  uint32_t* tbase = (uint32_t*)(bars + 16);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * kStage / 16; i += blockDim.x) ((uint4*)base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  long long cyc = 0;
  if (warp == 0) {
    const uint32_t idesc = umma_idesc_bf16(128, n);
    const uint32_t d = *tbase;
    const uint32_t ring = smem_u32(base);
    const uint64_t hi = umma_sdesc_sw128(0);
    const long long c0 = clock64();
    if (mode == 0) {
      uint32_t stage = 0, bits = 0;
      for (int k = 0; k < kb; ++k) {
        if (k >= lag) mbar_wait(&bars[stage], (bits >> stage) & 1u);
        if (!nofence) tc_fence_after();
        const uint32_t a0 = ring + stage * kStage, b0 = a0 + 16384;
        if (elect_one()) {
          umma_bf16(d, hi | ((a0 & 0x3FFFF) >> 4), hi | ((b0 & 0x3FFFF) >> 4), idesc, k > 0 ? 1u : 0u);
          umma_bf16(d, hi | (((a0 + 32) & 0x3FFFF) >> 4), hi | (((b0 + 32) & 0x3FFFF) >> 4), idesc, 1u);
          umma_bf16(d, hi | (((a0 + 64) & 0x3FFFF) >> 4), hi | (((b0 + 64) & 0x3FFFF) >> 4), idesc, 1u);
          umma_bf16(d, hi | (((a0 + 96) & 0x3FFFF) >> 4), hi | (((b0 + 96) & 0x3FFFF) >> 4), idesc, 1u);
          umma_commit(&bars[stage]);
        }
        __syncwarp();
        if (k >= lag) bits ^= 1u << stage;
        stage = stage + 1 == (uint32_t)lag ? 0 : stage + 1;
      }
    } else if (mode >= 3) {
      // whole warp; stages of 2 K blocks (8 MMAs): mode 3 = one wait + one commit per
      // stage, mode 4 = two waits + two commits per stage (one per K block, as mode 0)
      uint32_t stage = 0, bits = 0;
      for (int k = 0; k < kb; k += 2) {
        const int kk = k / 2;
        if (kk >= lag) mbar_wait(&bars[stage], (bits >> stage) & 1u);
        if ((mode == 4 || mode == 6) && kk >= lag) mbar_wait(&bars[stage + 4], (bits >> stage) & 1u);
        if (!nofence) tc_fence_after();
        const uint32_t a0 = ring + stage * kStage, b0 = a0 + 16384;
        if (elect_one()) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t ah = a0 + h * 8192, bh = b0 + h * 8192;
            umma_bf16(d, hi | ((ah & 0x3FFFF) >> 4), hi | ((bh & 0x3FFFF) >> 4), idesc, k + h > 0 ? 1u : 0u);
            umma_bf16(d, hi | (((ah + 32) & 0x3FFFF) >> 4), hi | (((bh + 32) & 0x3FFFF) >> 4), idesc, 1u);
            umma_bf16(d, hi | (((ah + 64) & 0x3FFFF) >> 4), hi | (((bh + 64) & 0x3FFFF) >> 4), idesc, 1u);
            umma_bf16(d, hi | (((ah + 96) & 0x3FFFF) >> 4), hi | (((bh + 96) & 0x3FFFF) >> 4), idesc, 1u);
            if ((mode == 4 || mode == 5 || mode == 6) && h == 0) umma_commit(&bars[stage + 4]);
          }
          umma_commit(&bars[stage]);
        }
        __syncwarp();
        if (kk >= lag) bits ^= 1u << stage;
        stage = stage + 1 == (uint32_t)lag ? 0 : stage + 1;
      }
    } else if (lane == 0) {
      uint32_t stage = 0, bits = 0;
      const uint64_t da_first = hi | ((ring & 0x3FFFF) >> 4);
      uint64_t da = da_first;
      for (int k = 0; k < kb; ++k) {
        if (k >= lag) mbar_wait(&bars[stage], (bits >> stage) & 1u);
        tc_fence_after();
        if (mode == 1) {
          const uint32_t a0 = ring + stage * kStage, b0 = a0 + 16384;
          umma_bf16(d, hi | ((a0 & 0x3FFFF) >> 4), hi | ((b0 & 0x3FFFF) >> 4), idesc, k > 0 ? 1u : 0u);
          umma_bf16(d, hi | (((a0 + 32) & 0x3FFFF) >> 4), hi | (((b0 + 32) & 0x3FFFF) >> 4), idesc, 1u);
          umma_bf16(d, hi | (((a0 + 64) & 0x3FFFF) >> 4), hi | (((b0 + 64) & 0x3FFFF) >> 4), idesc, 1u);
          umma_bf16(d, hi | (((a0 + 96) & 0x3FFFF) >> 4), hi | (((b0 + 96) & 0x3FFFF) >> 4), idesc, 1u);
        } else {
          const uint64_t db = da + (16384 >> 4);
          umma_bf16(d, da, db, idesc, k > 0 ? 1u : 0u);
          umma_bf16(d, da + 2, db + 2, idesc, 1u);
          umma_bf16(d, da + 4, db + 4, idesc, 1u);
          umma_bf16(d, da + 6, db + 6, idesc, 1u);
        }
        umma_commit(&bars[stage]);
        if (k >= lag) bits ^= 1u << stage;
        if (stage + 1 == (uint32_t)lag) {
          stage = 0;
          da = da_first;
        } else {
          ++stage;
          da += kStage >> 4;
        }
      }
    }
    __syncwarp();
    cyc = clock64() - c0;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = cyc;
  // drain: the last `lag` commits
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(*tbase, 512);
}

int main() {
  long long* d_out = nullptr;
  cudaMalloc(&d_out, 148 * sizeof(long long));
  cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kStage + 2048);
  printf("mode,nofence,n,lag,grid,cycles_per_kblock,tensor_frac\n");
  for (int mode : {0, 3, 4, 5, 6})
  for (int nofence : {0, 1})
    for (int n : {64, 128, 256})
      for (int lag : {2, 4})
        if (mode < 3 || n <= 128)
        for (int grid : {1, 148}) {
          const int kb = 4096;
          for (int w = 0; w < 2; ++w) mma_loop<<<grid, 128, 4 * kStage + 2048>>>(n, kb, lag, mode, nofence, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("cuda error %s\n", cudaGetErrorString(e));
            return 1;
          }
          std::vector<long long> o(grid);
          cudaMemcpy(o.data(), d_out, grid * sizeof(long long), cudaMemcpyDeviceToHost);
          double s = 0;
          for (auto v : o) s += (double)v;
          const double per = s / grid / kb;
          printf("%d,%d,%d,%d,%d,%.1f,%.3f\n", mode, nofence, n, lag, grid, per, 4 * (128.0 * n / 256) / per);
        }
  return 0;
}
