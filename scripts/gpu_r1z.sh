mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
for r in 1 2; do
GL_LIB=$D/libgpulet_base.so timeout 300 python tools/serve_ab.py --xs 0.5,1.0,2.0,3.0 --secs 0.5 > gpurun_out/ab_z_base_$r.log 2>&1
GL_LIB=$D/libgpulet_G.so timeout 300 python tools/serve_ab.py --xs 0.5,1.0,2.0,3.0 --secs 0.5 > gpurun_out/ab_z_G_$r.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_serve.py -m gpu -q > gpurun_out/gputests_r1z.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1z.log
timeout 600 python tools/consolidate.py --json gpurun_out/consolidate_b200.json > gpurun_out/consolidate_r1z.log 2>&1; echo "rc=$?" >> gpurun_out/consolidate_r1z.log
echo done
