# Epilogue residual prefetch + step prefetch + pack MLP: parity and per-step traces.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1d.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1d.log
for mb in resnet50:32 resnet50:8 vgg16:32 googlenet:32 ssd_mobilenet_v1:32 bert_base:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace_r1d_${m}_b${b}.json >> gpurun_out/oneshot_r1d.log 2>&1
done
timeout 600 python tools/gemm_micro.py --only res_l1_1x1_64,res_l1_1x1_256,res_l1_3x3_64,res_conv1,res_l3_3x3_256 --flags 0,2,12 --json gpurun_out/micro_r1d.json > gpurun_out/micro_r1d.log 2>&1
echo done
