mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_models.py -x -v -s > gpurun_out/models.log 2>&1; echo "models rc=$?" >> gpurun_out/models.log
dmesg 2>/dev/null | tail -5 >> gpurun_out/models.log
free -g >> gpurun_out/models.log
