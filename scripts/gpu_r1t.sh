mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1t.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1t.log
D=paper_2109_01611_b200/_ab
VARIANTS="base=$D/libgpulet_base.so F=$D/libgpulet_F.so" bash scripts/ab_oneshot.sh t resnet50:32 resnet50:15 resnet50:8 bert_base:32 bert_base:8 > gpurun_out/ab_t.log 2>&1
echo done
