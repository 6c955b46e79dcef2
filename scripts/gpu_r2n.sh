mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests_r2n.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2n.log
VARIANTS="P=$D/libgpulet_P.so Q=$D/libgpulet_Q.so" bash scripts/ab_oneshot.sh q resnet50:15 resnet50:8 resnet50:32 resnet50:1 googlenet:8 googlenet:15 ssd_mobilenet_v1:8 vgg16:8 bert_base:8 > gpurun_out/ab_q.log 2>&1
echo done
