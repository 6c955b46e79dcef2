mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/exec9.log 2>&1; echo "exec rc=$?" >> gpurun_out/exec9.log
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or conv" > gpurun_out/kern9.log 2>&1; echo "kern rc=$?" >> gpurun_out/kern9.log
timeout 300 python -m pytest tests/test_gpu_models.py -q -x > gpurun_out/models9.log 2>&1; echo "models rc=$?" >> gpurun_out/models9.log
for mb in resnet50:1 resnet50:32 vgg16:32 bert_base:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace9_${m}_b${b}.json >> gpurun_out/oneshot9.log 2>&1
done
