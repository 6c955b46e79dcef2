mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_r2w.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2w.log
for r in 1 2; do
GL_LIB=$D/libgpulet_base.so timeout 600 python tools/latency_ab.py >> gpurun_out/lat_w.log 2>&1
GL_LIB=$D/libgpulet_S.so timeout 600 python tools/latency_ab.py >> gpurun_out/lat_w.log 2>&1
done
echo done
