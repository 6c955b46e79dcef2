mkdir -p gpurun_out
for bn in 0 64 128 256; do for mb in resnet50:15 resnet50:8 googlenet:15 ssd_mobilenet_v1:8; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --bn $bn --json gpurun_out/bn_${bn}_${m}_b${b}.json > /dev/null 2>&1
done; done
echo done
