mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/gputests_r2g.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2g.log
VARIANTS="J=$D/libgpulet_J.so L=$D/libgpulet_L.so" bash scripts/ab_oneshot.sh g googlenet:8 googlenet:15 googlenet:32 resnet50:8 resnet50:15 ssd_mobilenet_v1:8 bert_base:8 > gpurun_out/ab_g.log 2>&1
echo done
