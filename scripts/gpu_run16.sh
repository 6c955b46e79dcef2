mkdir -p gpurun_out
timeout 600 python tools/gemm_micro.py --bn 0,64,128,256 --json gpurun_out/micro16.json > gpurun_out/micro16.log 2>&1
for mb in resnet50:32 vgg16:32 bert_base:32 googlenet:32 ssd_mobilenet_v1:32 resnet50:1; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace16_${m}_b${b}.json >> gpurun_out/oneshot16.log 2>&1
done
