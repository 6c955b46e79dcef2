"""gpu-let serving hot path for B200 (arXiv 2109.01611), native library + thin binding.

The product is `libgpulet.so` (csrc/: CUDA executor and layer kernels for
sm_100a, runtime, program builders, scheduler) behind include/gpulet.h; the
Python module `gpulet` only marshals arguments.
"""
from . import gpulet  # noqa: F401
