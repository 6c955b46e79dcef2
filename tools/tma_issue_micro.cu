// TMA issue-cost microbenchmark (tuning tool, not part of the product).
// One CTA per SM; one thread issues `n` 2-D tiled TMA loads back to back into
// `n` distinct shared-memory slots (no waits between issues), each with its own
// mbarrier, then waits for all of them.  Reports SM cycles of the issue loop
// alone and of issue + completion, per load, for
//   map = 0: tensor map passed as a __grid_constant__ kernel parameter,
//   map = 1: tensor map in global memory, prefetched (prefetch.tensormap),
//   map = 2: tensor map in global memory, not prefetched,
// and box heights of 8 .. 256 rows x 64 bf16 (128-B swizzle), L2-resident source.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2109_01611_b200/csrc \
//        tools/tma_issue_micro.cu -o tools/tma_issue_micro -lcuda && ./tools/tma_issue_micro
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

__global__ void __launch_bounds__(32, 1) tma_issue(const __grid_constant__ CUtensorMap pmap, const CUtensorMap* gmap,
                                                   int mode, int rows, int n, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(base + 196608);
  const void* map = mode == 0 ? (const void*)&pmap : (const void*)gmap;
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    if (mode == 1) asm volatile("prefetch.tensormap [%0];" ::"l"(gmap) : "memory");
  }
  __syncwarp();
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)rows * 128;
    // warm-up load (descriptor fetch) into slot 0, waited
    mbar_arrive_expect_tx(&bars[0], bytes);
    tma_load_2d(smem_u32(base), map, &bars[0], 0, 0);
    mbar_wait(&bars[0], 0);
    const long long c0 = clock64();
    for (int i = 0; i < n; ++i) {
      mbar_arrive_expect_tx(&bars[i], bytes);
      tma_load_2d(smem_u32(base + (uint32_t)i * bytes), map, &bars[i], (i & 7) * 64, (blockIdx.x * 8 + i) * rows);
    }
    const long long c1 = clock64();
    for (int i = 0; i < n; ++i) mbar_wait(&bars[i], i == 0 ? 1 : 0);
    const long long c2 = clock64();
    out[2 * blockIdx.x] = c1 - c0;
    out[2 * blockIdx.x + 1] = c2 - c0;
  }
}

// Steady state, one thread, ring of `depth` slots, `iters` loads:
//   batched = 0: per load, wait for the slot's previous load, then re-arm and issue;
//   batched = 1: issue `depth` loads, then wait for all of them, repeat.
__global__ void __launch_bounds__(32, 1) tma_steady(const CUtensorMap* gmap, int rows, int depth, int iters,
                                                    int batched, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(base + 196608);
  if (threadIdx.x != 0) return;
  for (int i = 0; i < depth; ++i) mbar_init(&bars[i], 1);
  fence_mbar_init();
  asm volatile("prefetch.tensormap [%0];" ::"l"(gmap) : "memory");
  const uint32_t bytes = (uint32_t)rows * 128;
  const long long c0 = clock64();
  if (!batched) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % depth;
      if (i >= depth) mbar_wait(&bars[s], ((i / depth) - 1) & 1);
      mbar_arrive_expect_tx(&bars[s], bytes);
      tma_load_2d(smem_u32(base + (uint32_t)s * bytes), gmap, &bars[s], (i & 7) * 64, ((blockIdx.x * 8 + s) * rows) & 16383);
    }
    for (int i = iters - depth; i < iters; ++i) mbar_wait(&bars[i % depth], (i / depth) & 1);
  } else if (batched == 2) {   // per slot wait, then two loads on the slot's barrier (2-K-block stages)
    for (int i = 0; i < iters; i += 2) {
      const int j = i / 2, s = j % depth;
      if (j >= depth) mbar_wait(&bars[s], ((j / depth) - 1) & 1);
      mbar_arrive_expect_tx(&bars[s], 2 * bytes);
      tma_load_2d(smem_u32(base + (uint32_t)s * bytes), gmap, &bars[s], (i & 7) * 64, ((blockIdx.x * 8 + s) * rows) & 16383);
      tma_load_2d(smem_u32(base + (uint32_t)s * bytes), gmap, &bars[s], ((i + 1) & 7) * 64, ((blockIdx.x * 8 + s) * rows) & 16383);
    }
    for (int j = iters / 2 - depth; j < iters / 2; ++j) mbar_wait(&bars[j % depth], (j / depth) & 1);
  } else {
    for (int g = 0; g < iters / depth; ++g) {
      for (int s = 0; s < depth; ++s) {
        mbar_arrive_expect_tx(&bars[s], bytes);
        tma_load_2d(smem_u32(base + (uint32_t)s * bytes), gmap, &bars[s], (s & 7) * 64, ((blockIdx.x * 8 + s) * rows) & 16383);
      }
      for (int s = 0; s < depth; ++s) mbar_wait(&bars[s], g & 1);
    }
  }
  out[blockIdx.x] = clock64() - c0;
}

int main() {
  const int64_t cols = 512, total_rows = 1 << 14;   // 16 MiB bf16 (L2-resident after the first pass)
  void* mat = nullptr;
  cudaMalloc(&mat, (size_t)cols * total_rows * 2);
  cudaMemset(mat, 1, (size_t)cols * total_rows * 2);
  long long* d_out = nullptr;
  cudaMalloc(&d_out, 2 * 148 * sizeof(long long));
  CUtensorMap* d_map = nullptr;
  cudaMalloc(&d_map, sizeof(CUtensorMap));
  cudaFuncSetAttribute(tma_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
  printf("mode,rows,n,grid,issue_cyc_per_load,total_cyc_per_load\n");
  for (int rows : {8, 32, 64, 128, 256}) {
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
    cudaMemcpy(d_map, &map, sizeof(map), cudaMemcpyHostToDevice);
    for (int mode : {0, 1, 2})
      for (int n : {1, 2, 4, 8, 16})
        for (int grid : {1, 148}) {
          if ((size_t)n * rows * 128 > 196608) continue;
          for (int w = 0; w < 3; ++w) tma_issue<<<grid, 32, 196608 + 2048>>>(map, d_map, mode, rows, n, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("cuda error %s\n", cudaGetErrorString(e));
            return 1;
          }
          std::vector<long long> o(2 * grid);
          cudaMemcpy(o.data(), d_out, 2 * grid * sizeof(long long), cudaMemcpyDeviceToHost);
          double a = 0, b = 0;
          for (int i = 0; i < grid; ++i) a += (double)o[2 * i], b += (double)o[2 * i + 1];
          printf("%d,%d,%d,%d,%.1f,%.1f\n", mode, rows, n, grid, a / grid / n, b / grid / n);
        }
  }
  printf("# steady: rows,depth,batched,grid,cyc_per_load\n");
  for (int rows : {64, 128, 256}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)total_rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(d_map, &map, sizeof(map), cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(tma_steady, cudaFuncAttributeMaxDynamicSharedMemorySize, 196608 + 2048);
    for (int depth : {2, 4, 8})
      for (int batched : {0, 1, 2})
        for (int grid : {1, 148}) {
          if ((size_t)depth * rows * 128 > 196608) continue;
          const int iters = 2048;
          for (int w = 0; w < 2; ++w) tma_steady<<<grid, 32, 196608 + 2048>>>(d_map, rows, depth, iters, batched, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("cuda error %s\n", cudaGetErrorString(e));
            return 1;
          }
          std::vector<long long> o(grid);
          cudaMemcpy(o.data(), d_out, grid * sizeof(long long), cudaMemcpyDeviceToHost);
          double a = 0;
          for (int i = 0; i < grid; ++i) a += (double)o[i];
          printf("steady,%d,%d,%d,%d,%.1f\n", rows, depth, batched, grid, a / grid / iters);
        }
  }
  return 0;
}
