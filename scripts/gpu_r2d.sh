mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
VARIANTS="I=$D/libgpulet_I.so J=$D/libgpulet_J.so" bash scripts/ab_oneshot.sh d googlenet:8 googlenet:32 resnet50:15 ssd_mobilenet_v1:8 bert_base:8 > gpurun_out/ab_d.log 2>&1
timeout 600 python -m pytest tests/test_gpu_models.py tests/test_gpu_serve.py -m gpu -q > gpurun_out/gputests_r2d.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2d.log
echo done
