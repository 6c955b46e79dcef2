mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/gputests21.log 2>&1; echo "rc=$?" >> gpurun_out/gputests21.log
timeout 600 python tools/gemm_micro.py --flags 0,8,12 --json gpurun_out/micro21.json > gpurun_out/micro21.log 2>&1
for mb in resnet50:32 vgg16:32 bert_base:32 googlenet:32 ssd_mobilenet_v1:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace21_${m}_b${b}.json >> gpurun_out/oneshot21.log 2>&1
done
