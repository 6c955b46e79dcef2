mkdir -p gpurun_out
for b in 18 19 20 21 22 23 24 25 26; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_resnet50_b$b.csv python tools/oneshot.py --model resnet50 --batch $b --reps 3 > /dev/null 2>&1
done
echo done
