mkdir -p gpurun_out
for sp in 0 2 4 8 16; do for mb in resnet50:15 resnet50:8 bert_base:8 vgg16:8; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --split $sp --json gpurun_out/sp_${sp}_${m}_b${b}.json > /dev/null 2>&1
done; done
echo done
