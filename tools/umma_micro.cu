// tcgen05.mma issue / execution microbenchmark (tuning tool, not part of the
// product): one CTA per SM, one elected thread issues `kb` K blocks of 4
// tcgen05.mma.cta_group::1.kind::f16 (M = 128, N in {64, 128, 256}, K = 16
// each, operands in 128-B-swizzled shared memory) and commits each K block to
// an mbarrier, waiting for the commit `lag` K blocks later (a ring of `lag`
// stages, as the executor's MMA warp does).  Reports ns per K block per CTA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2109_01611_b200/csrc \
//        tools/umma_micro.cu -o tools/umma_micro && ./tools/umma_micro
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

__global__ void __launch_bounds__(256, 1) umma_loop(int n, int kb, int lag, int nw, int alt, uint64_t* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(base + 4 * 49152);   // [4 warps][8]
  uint32_t* tbase = (uint32_t*)(bars + 40);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4 * 49152 / 16; i += blockDim.x) ((uint4*)base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 32; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (warp == 7) tmem_alloc(tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  uint64_t t0 = globaltimer();
  const long long c0 = clock64();
  if (warp < nw) {   // warp w issues into its own accumulator (512 / nw columns apart)
    const uint32_t idesc = umma_idesc_bf16(128, n);
    const uint32_t d = *tbase + (uint32_t)warp * (512 / nw);  // alt accumulators of n columns inside
    uint64_t* bars_w = bars + warp * 8;
    // lag 0: no per-K-block commit / wait at all (one commit at the end): the
    // tensor pipe's own rate for back-to-back tcgen05.mma from one thread
    const int L = lag > 0 ? lag : 1;
    for (int k = 0; k < kb; ++k) {
      const int s = k % L;
      if (lag > 0 && k >= lag) mbar_wait(&bars_w[s], ((k / lag) - 1) & 1);
      if (elect_one()) {
        const uint32_t a0 = smem_u32(base + s * 49152), b0 = a0 + 16384;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          umma_bf16(d + (uint32_t)((j % alt) * n), umma_sdesc_sw128(a0 + 32 * j), umma_sdesc_sw128(b0 + 32 * j), idesc,
                    k > 0 || j >= alt ? 1u : 0u);
        if (lag > 0 || k == kb - 1) umma_commit(&bars_w[s]);
      }
      __syncwarp();
    }
    if (lag == 0) mbar_wait(&bars_w[0], 0);
    for (int k = kb - lag; lag > 0 && k < kb; ++k)
      if (k >= 0) mbar_wait(&bars_w[k % lag], (k / lag) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out_ns[blockIdx.x] = globaltimer() - t0;
    out_ns[gridDim.x + blockIdx.x] = (uint64_t)(clock64() - c0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 7) tmem_dealloc(*tbase, 512);
}

int main() {
  uint64_t* d_ns = nullptr;
  cudaMalloc(&d_ns, 2 * 148 * sizeof(uint64_t));
  cudaFuncSetAttribute(umma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("n,lag,grid,issuing_warps,alt_accumulators,ns_per_kblock_per_warp,cycles_per_umma_per_warp,tensor_frac_sm\n");
  for (int n : {64, 128, 256})
    for (int lag : {0, 2, 4})
      for (int nw : {1, 2, 4})
      for (int alt : {1, 2, 4})
      for (int grid : {1, 148}) {
        if (n * nw * alt > 512) continue;
        const int kb = 4096;
        for (int w = 0; w < 2; ++w) umma_loop<<<grid, 256, 200 * 1024>>>(n, kb, lag, nw, alt, d_ns);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("cuda error %s\n", cudaGetErrorString(e));
          return 1;
        }
        std::vector<uint64_t> ns(2 * grid);
        cudaMemcpy(ns.data(), d_ns, 2 * grid * sizeof(uint64_t), cudaMemcpyDeviceToHost);
        double sum = 0, csum = 0;
        for (int i = 0; i < grid; ++i) sum += (double)ns[i], csum += (double)ns[grid + i];
        const double per = sum / grid / kb;
        const double cyc = csum / grid / kb / 4;                 // SM clock cycles per UMMA (clock64)
        const double floor_cyc = 128.0 * n / 256;               // tcgen05 floor, M = 128, cta_group::1
        printf("%d,%d,%d,%d,%d,%.1f,%.1f,%.3f\n", n, lag, grid, nw, alt, per, cyc, nw * floor_cyc / cyc);
      }
  return 0;
}
