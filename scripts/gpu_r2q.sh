mkdir -p gpurun_out
export GL_BENCH_WATCHDOG_S=1400
timeout 1500 python bench.py --verbose > gpurun_out/bench_r2q.json 2> gpurun_out/bench_r2q.err; echo "rc=$?" >> gpurun_out/bench_r2q.err
for mb in resnet50:14 resnet50:13 resnet50:12; do m=${mb%:*}; b=${mb#*:}
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_${m}_b$b.csv python tools/oneshot.py --model $m --batch $b --reps 3 > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/ncu_traffic_${m}_b$b.csv $m $b >> gpurun_out/oneshot_r2q.log 2>&1
done
cp profiles/ncu_*.json gpurun_out/ 2>/dev/null
timeout 600 python tools/adapt.py --json gpurun_out/adapt_b200.json > gpurun_out/adapt_r2q.log 2>&1
echo done
