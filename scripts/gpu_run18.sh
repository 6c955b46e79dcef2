mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests18.log 2>&1; echo "rc=$?" >> gpurun_out/gputests18.log
for mb in resnet50:32 vgg16:32 bert_base:32 googlenet:32 ssd_mobilenet_v1:32 resnet50:1 lenet5:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace18_${m}_b${b}.json >> gpurun_out/oneshot18.log 2>&1
done
