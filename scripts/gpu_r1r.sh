mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
for r in 1 2; do
GL_LIB=$D/libgpulet_base.so timeout 300 python tools/serve_ab.py --xs 1.5,2.0,2.5,3.0 --secs 0.5 > gpurun_out/ab_r_base_$r.log 2>&1
GL_LIB=$D/libgpulet_E.so timeout 300 python tools/serve_ab.py --xs 1.5,2.0,2.5,3.0 --secs 0.5 > gpurun_out/ab_r_E_$r.log 2>&1
GL_SERVE_NO_RT=1 GL_LIB=$D/libgpulet_E.so timeout 300 python tools/serve_ab.py --xs 1.5,2.0,2.5,3.0 --secs 0.5 > gpurun_out/ab_r_Enort_$r.log 2>&1
done
timeout 300 python -m pytest tests/test_gpu_models.py tests/test_gpu_serve.py -m gpu -q -x > gpurun_out/gputests_r1r.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1r.log
echo done
