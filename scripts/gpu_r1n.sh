mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_executor.py -m gpu -q -x > gpurun_out/gputests_r1n.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1n.log
D=paper_2109_01611_b200/_ab
VARIANTS="C1=$D/libgpulet_C1.so D2=$D/libgpulet_D2.so" bash scripts/ab_oneshot.sh n resnet50:32 resnet50:8 bert_base:32 googlenet:8 > gpurun_out/ab_n.log 2>&1
echo done
