// tcgen05.mma issue-rate microbenchmark with loop-invariant operands (tuning
// tool, not part of the product).  One CTA per SM; `nw` warps, one elected
// thread each, issue `iters` x 4 tcgen05.mma.cta_group::1.kind::f16
// (M = 128, N in {64, 128, 256}, K = 16) whose shared-memory descriptors are
// computed once before the loop (4 K steps of one 128-B-swizzled stage), into
// its own accumulator, one commit at the end.  Reports SM cycles per MMA per
// issuing thread and the CTA's fraction of the cta_group::1 tensor floor
// (128 x N / 256 cycles per MMA).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2109_01611_b200/csrc \
//        tools/umma_issue_micro.cu -o tools/umma_issue_micro && ./tools/umma_issue_micro
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

__global__ void __launch_bounds__(128, 1) umma_issue(int n, int iters, int nw, int variant, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(base + 65536);
  uint32_t* tbase = (uint32_t*)(bars + 12);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) ((uint4*)base)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  fence_proxy_async_smem();
  long long cyc = 0;
  if (warp < nw) {
    const uint32_t idesc = umma_idesc_bf16(128, n);
    const uint32_t d = *tbase + (uint32_t)warp * (512 / nw);
    const uint32_t a0 = smem_u32(base), b0 = a0 + 16384;
    const uint64_t da0 = umma_sdesc_sw128(a0), da1 = umma_sdesc_sw128(a0 + 32), da2 = umma_sdesc_sw128(a0 + 64),
                   da3 = umma_sdesc_sw128(a0 + 96);
    const uint64_t db0 = umma_sdesc_sw128(b0), db1 = umma_sdesc_sw128(b0 + 32), db2 = umma_sdesc_sw128(b0 + 64),
                   db3 = umma_sdesc_sw128(b0 + 96);
    __syncwarp();
    const long long c0 = clock64();
    if (variant > 0) {
      // the whole warp walks the loop, one elected lane issues each group of 4:
      // 1 = loop-invariant descriptors; 2 = + a commit per group (no wait);
      // 3 = descriptors rebuilt per group from a rotating stage address (4 stages)
      const uint64_t hi = umma_sdesc_sw128(0);
#pragma unroll 1
      for (int k = 0; k < iters; ++k) {
        // stage stride 0 at run time (iters < 2^30), unknown to the compiler
        const uint32_t st = (uint32_t)k & 3u, stride = (uint32_t)(iters >> 30) * 16384u;
        if (elect_one()) {
          if (variant == 3) {
            const uint32_t ra = a0 + st * stride, rb = b0 + st * stride;
            umma_bf16(d, hi | ((ra & 0x3FFFF) >> 4), hi | ((rb & 0x3FFFF) >> 4), idesc, k > 0 ? 1u : 0u);
            umma_bf16(d, hi | (((ra + 32) & 0x3FFFF) >> 4), hi | (((rb + 32) & 0x3FFFF) >> 4), idesc, 1u);
            umma_bf16(d, hi | (((ra + 64) & 0x3FFFF) >> 4), hi | (((rb + 64) & 0x3FFFF) >> 4), idesc, 1u);
            umma_bf16(d, hi | (((ra + 96) & 0x3FFFF) >> 4), hi | (((rb + 96) & 0x3FFFF) >> 4), idesc, 1u);
          } else {
            umma_bf16(d, da0, db0, idesc, k > 0 ? 1u : 0u);
            umma_bf16(d, da1, db1, idesc, 1u);
            umma_bf16(d, da2, db2, idesc, 1u);
            umma_bf16(d, da3, db3, idesc, 1u);
          }
          if (variant == 2) umma_commit(&bars[4 + (k & 3)]);
        }
        __syncwarp();
      }
      if (elect_one()) umma_commit(&bars[warp]);
    } else if (elect_one()) {
      umma_bf16(d, da0, db0, idesc, 0u);
      umma_bf16(d, da1, db1, idesc, 1u);
      umma_bf16(d, da2, db2, idesc, 1u);
      umma_bf16(d, da3, db3, idesc, 1u);
#pragma unroll 1
      for (int k = 1; k < iters; ++k) {
        umma_bf16(d, da0, db0, idesc, 1u);
        umma_bf16(d, da1, db1, idesc, 1u);
        umma_bf16(d, da2, db2, idesc, 1u);
        umma_bf16(d, da3, db3, idesc, 1u);
      }
      umma_commit(&bars[warp]);
    }
    __syncwarp();
    mbar_wait(&bars[warp], 0);
    cyc = clock64() - c0;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && warp < nw) out[blockIdx.x * 4 + warp] = cyc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(*tbase, 512);
}

int main() {
  long long* d_out = nullptr;
  cudaMalloc(&d_out, 4 * 148 * sizeof(long long));
  cudaFuncSetAttribute(umma_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
  printf("variant,n,issuing_warps,grid,cycles_per_umma_per_thread,tensor_frac_sm\n");
  for (int variant : {0, 1, 2, 3})
  for (int n : {64, 128, 256})
    for (int nw : {1, 2, 4})
      for (int grid : {1, 148}) {
        if (n * nw > 512 || (variant > 0 && nw > 1)) continue;
        const int iters = 4096;
        for (int w = 0; w < 2; ++w) umma_issue<<<grid, 128, 65536 + 2048>>>(n, iters, nw, variant, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("cuda error %s\n", cudaGetErrorString(e));
          return 1;
        }
        std::vector<long long> o(4 * grid);
        cudaMemcpy(o.data(), d_out, 4 * grid * sizeof(long long), cudaMemcpyDeviceToHost);
        double s = 0;
        for (int b = 0; b < grid; ++b)
          for (int w = 0; w < nw; ++w) s += (double)o[4 * b + w];
        const double cyc = s / (grid * nw) / (4.0 * iters);
        printf("%d,%d,%d,%d,%.1f,%.3f\n", variant, n, nw, grid, cyc, nw * (128.0 * n / 256) / cyc);
      }
  return 0;
}
