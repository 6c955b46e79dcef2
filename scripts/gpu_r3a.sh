mkdir -p gpurun_out
A=paper_2109_01611_b200/_ab
timeout 600 python -m pytest tests -m gpu -q -k "lenet" > gpurun_out/gputests_r3a.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r3a.log
VARIANTS="base=$A/libgpulet_base.so lenet=$A/libgpulet_lenet.so" timeout 900 bash scripts/ab_oneshot.sh r3a lenet5:1 lenet5:8 lenet5:32 resnet50:15 > gpurun_out/ab_r3a.log 2>&1
for rep in 1 2; do for v in base lenet; do
  GL_LIB=$A/libgpulet_$v.so timeout 300 python tools/latency_ab.py > gpurun_out/lat_r3a_${v}_$rep.log 2>&1
  GL_LIB=$A/libgpulet_$v.so timeout 300 python tools/serve_ab.py --xs 1.9,2.27,2.6 --secs 0.5 > gpurun_out/serve_r3a_${v}_$rep.log 2>&1
done; done
echo done
