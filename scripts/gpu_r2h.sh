mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_fullsize.py tests/test_gpu_kernels.py -m gpu -q -x > gpurun_out/gputests_r2h.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2h.log
VARIANTS="L=$D/libgpulet_L.so M=$D/libgpulet_M.so" bash scripts/ab_oneshot.sh h resnet50:8 resnet50:15 resnet50:32 resnet50:1 bert_base:8 bert_base:32 ssd_mobilenet_v1:8 googlenet:8 vgg16:8 vgg16:1 > gpurun_out/ab_h.log 2>&1
echo done
