mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r2e.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2e.log
VARIANTS="J=$D/libgpulet_J.so K=$D/libgpulet_K.so" bash scripts/ab_oneshot.sh e resnet50:15 resnet50:32 resnet50:1 googlenet:8 bert_base:8 vgg16:8 > gpurun_out/ab_e.log 2>&1
echo done
