mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests_r2j.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2j.log
VARIANTS="L=$D/libgpulet_L.so N=$D/libgpulet_N.so" bash scripts/ab_oneshot.sh j resnet50:8 resnet50:15 resnet50:1 bert_base:8 ssd_mobilenet_v1:8 googlenet:8 > gpurun_out/ab_j.log 2>&1
echo done
