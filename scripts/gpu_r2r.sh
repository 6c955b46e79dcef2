mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py -m gpu -q > gpurun_out/gputests_r2r.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2r.log
VARIANTS="P=$D/libgpulet_P.so R=$D/libgpulet_R.so" bash scripts/ab_oneshot.sh r resnet50:15 resnet50:32 googlenet:15 vgg16:8 bert_base:8 > gpurun_out/ab_r2.log 2>&1
echo done
