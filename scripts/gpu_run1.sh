set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -40 | tee gpurun_out/kern.log
timeout 600 python -m pytest tests/test_gpu_executor.py -x -q 2>&1 | tail -30 | tee gpurun_out/exec.log
