mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1m.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1m.log
D=paper_2109_01611_b200/_ab
VARIANTS="C1=$D/libgpulet_C1.so D=$D/libgpulet_D.so" bash scripts/ab_oneshot.sh m resnet50:32 resnet50:8 resnet50:15 bert_base:32 googlenet:8 ssd_mobilenet_v1:8 > gpurun_out/ab_m.log 2>&1
echo done
