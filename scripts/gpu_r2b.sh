mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
for r in 1 2 3; do
GL_LIB=$D/libgpulet_I.so timeout 300 python tools/latency_ab.py >> gpurun_out/lat_ab2.log 2>&1
GL_LIB=$D/libgpulet_I.so timeout 300 python tools/latency_ab.py >> gpurun_out/lat_ab2.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_executor.py tests/test_gpu_serve.py tests/test_gpu_models.py -m gpu -q > gpurun_out/gputests_r2b.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2b.log
echo done
