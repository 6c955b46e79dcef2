mkdir -p gpurun_out
A=paper_2109_01611_b200/_ab
VARIANTS="lenet=$A/libgpulet_lenet.so fc4=$A/libgpulet_fc4.so" timeout 600 bash scripts/ab_oneshot.sh r3b lenet5:1 lenet5:24 > gpurun_out/ab_r3b.log 2>&1
for v in lenet fc4; do GL_LIB=$A/libgpulet_$v.so timeout 300 python tools/latency_ab.py > gpurun_out/lat_r3b_${v}.log 2>&1; done
bash scripts/measure_all.sh r3b
echo done
