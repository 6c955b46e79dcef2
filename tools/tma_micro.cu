// TMA load pipeline microbenchmark (tuning tool, not part of the product):
// one CTA per SM, one producer thread streaming 2-D tiled TMA boxes of
// `rows` x 64 bf16 (128-B swizzle, as the executor's GEMM operands) through a
// ring of `depth` stages, one consumer thread that waits each stage's full
// barrier and frees it at once (no math).  Reports ns per stage per CTA and
// the aggregate GB/s for grids of 1 and 148 CTAs and depths 1..8, with the
// source matrix L2-resident (re-read) or streamed from HBM (fresh rows).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2109_01611_b200/csrc \
//        tools/tma_micro.cu -o tools/tma_micro -lcuda && ./tools/tma_micro
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

// Non-suspending spin on an mbarrier phase (mbarrier.test_wait), to compare with
// mbar_wait's try_wait loop (which may suspend the thread until a time limit).
__device__ __forceinline__ void spin_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void wait_any(uint64_t* bar, uint32_t parity, int spin) {
  if (spin) spin_wait(bar, parity);
  else mbar_wait(bar, parity);
}

__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap map, int rows, int depth,
                                                    int iters, int row_span, int spin, uint64_t* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + 196608);
  uint64_t* empty = full + 8;
  const uint32_t stage_bytes = (uint32_t)rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < depth; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t t0 = globaltimer();
  if (threadIdx.x == 0) {          // producer
    for (int i = 0; i < iters; ++i) {
      const int s = i % depth;
      wait_any(&empty[s], ((i / depth) & 1) ^ 1, spin);
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      const int row = (blockIdx.x * iters + i) * rows % row_span;
      tma_load_2d(smem_u32(base + s * stage_bytes), &map, &full[s], (i & 7) * 64, row);
    }
  } else if (threadIdx.x == 32) {  // consumer
    for (int i = 0; i < iters; ++i) {
      const int s = i % depth;
      wait_any(&full[s], (i / depth) & 1, spin);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out_ns[blockIdx.x] = globaltimer() - t0;
}

// Producer-only variants: mode 1 = one thread, waits its own stage's previous
// load (no consumer hop); mode 2 = `nprod` warps, warp w owns stages w, w+nprod, ...
__global__ void __launch_bounds__(128, 1) tma_self(const __grid_constant__ CUtensorMap map, int rows, int depth,
                                                  int iters, int row_span, int nprod, uint64_t* out_ns) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(base + 196608);
  const uint32_t stage_bytes = (uint32_t)rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < depth; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t t0 = globaltimer();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0 && w < nprod) {
    for (int i = w; i < iters; i += nprod) {
      const int s = i % depth;
      if (i >= depth) mbar_wait(&full[s], ((i / depth) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], stage_bytes);
      const int row = (blockIdx.x * iters + i) * rows % row_span;
      tma_load_2d(smem_u32(base + s * stage_bytes), &map, &full[s], (i & 7) * 64, row);
    }
    for (int i = iters - depth + w; i < iters; i += nprod)
      if (i >= 0) mbar_wait(&full[i % depth], (i / depth) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out_ns[blockIdx.x] = globaltimer() - t0;
}

int main() {
  const int64_t cols = 512, total_rows = 1 << 17;      // 128 MiB bf16 matrix (512 columns)
  void* mat = nullptr;
  cudaMalloc(&mat, (size_t)cols * total_rows * 2);
  cudaMemset(mat, 1, (size_t)cols * total_rows * 2);
  uint64_t* d_ns = nullptr;
  cudaMalloc(&d_ns, 148 * sizeof(uint64_t));
  cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
  printf("rows,stage_kb,depth,grid,span,spin,ns_per_stage_per_cta,agg_gbs\n");
  for (int rows : {64, 128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)total_rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    if (cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    for (int span : {4096, 1 << 17}) {   // 4 MiB window (L2-resident) or the whole 128 MiB (HBM)
      for (int grid : {1, 148}) {
        for (int depth : {1, 2, 4, 6, 8})
        for (int spin : {0, 1}) {
          if (depth * rows * 128 > 196608) continue;
          const int iters = 2048;
          for (int w = 0; w < 2; ++w)
            tma_stream<<<grid, 64, 196608 + 2048>>>(map, rows, depth, iters, span, spin, d_ns);
          cudaDeviceSynchronize();
          std::vector<uint64_t> ns(grid);
          cudaMemcpy(ns.data(), d_ns, grid * sizeof(uint64_t), cudaMemcpyDeviceToHost);
          uint64_t mx = 0;
          double sum = 0;
          for (auto v : ns) mx = v > mx ? v : mx, sum += (double)v;
          const double per = sum / grid / iters;
          const double gbs = (double)grid * iters * rows * 128 / (double)mx;
          printf("%d,%d,%d,%d,%d,%d,%.1f,%.1f\n", rows, rows * 128 / 1024, depth, grid, span, spin, per, gbs);
        }
      }
    }
  }
  cudaFuncSetAttribute(tma_self, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
  printf("# producer-only: rows,depth,grid,nprod,ns_per_stage_per_cta,agg_gbs\n");
  for (int rows : {128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)total_rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int grid : {1, 148})
      for (int depth : {4, 6, 8})
        for (int nprod : {1, 2, 4}) {
          if (depth * rows * 128 > 196608 || depth % nprod) continue;
          const int iters = 2048;
          for (int w = 0; w < 2; ++w)
            tma_self<<<grid, 128, 196608 + 2048>>>(map, rows, depth, iters, 4096, nprod, d_ns);
          cudaDeviceSynchronize();
          std::vector<uint64_t> ns(grid);
          cudaMemcpy(ns.data(), d_ns, grid * sizeof(uint64_t), cudaMemcpyDeviceToHost);
          uint64_t mx = 0;
          double sum = 0;
          for (auto v : ns) mx = v > mx ? v : mx, sum += (double)v;
          printf("self,%d,%d,%d,%d,%.1f,%.1f\n", rows, depth, grid, nprod, sum / grid / iters,
                 (double)grid * iters * rows * 128 / (double)mx);
        }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("cuda error %s\n", cudaGetErrorString(e));
  return 0;
}
