// K12: HBM bandwidth probe confined to a gpu-let's SMs ("BW(n)
// is *measured* by K12 (a stream copy inside the same green context)"; the
// per-gpu-let HBM roof of the metric "per-gpu-let tensor/HBM % of roofline").
// A plain grid-stride copy with 16-B loads, four loads in flight per thread,
// launched on the green-context stream of the gpu-let size under test
// (runtime.cpp gl_bw_probe); n SMs need not saturate HBM, which is what the
// probe measures.
#include <cuda_runtime.h>

#include <cstdint>

namespace {
__global__ void __launch_bounds__(512) bw_copy(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const int4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
               d = __ldcs(src + i + 3 * stride);
    __stcs(dst + i, a);
    __stcs(dst + i + stride, b);
    __stcs(dst + i + 2 * stride, c);
    __stcs(dst + i + 3 * stride, d);
  }
  for (; i < n; i += stride) __stcs(dst + i, __ldcs(src + i));
}
}  // namespace

extern "C" cudaKernel_t gl_probe_handle() {
  cudaKernel_t k = nullptr;
  if (cudaGetKernel(&k, (const void*)bw_copy) != cudaSuccess) return nullptr;
  return k;
}
