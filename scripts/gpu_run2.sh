set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_executor.py -x -q 2>&1 | tail -30 | tee gpurun_out/exec.log
timeout 900 python -m pytest tests/test_gpu_models.py -x -q 2>&1 | tail -40 | tee gpurun_out/models.log
