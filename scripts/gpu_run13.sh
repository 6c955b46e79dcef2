mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/exec13.log 2>&1; echo "exec rc=$?" >> gpurun_out/exec13.log
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kern13.log 2>&1; echo "kern rc=$?" >> gpurun_out/kern13.log
timeout 300 python -m pytest tests/test_gpu_models.py -q -x > gpurun_out/models13.log 2>&1; echo "models rc=$?" >> gpurun_out/models13.log
for mb in resnet50:1 resnet50:32 vgg16:32 bert_base:32 googlenet:32 ssd_mobilenet_v1:32 lenet5:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace13_${m}_b${b}.json >> gpurun_out/oneshot13.log 2>&1
done
