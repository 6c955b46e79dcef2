# Full round measurement after the epilogue/prefetch/frontend changes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1h.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1h.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r1h.log
export GL_BENCH_WATCHDOG_S=1100
timeout 1200 python bench.py --verbose > gpurun_out/bench_r1h.json 2> gpurun_out/bench_r1h.err; echo "rc=$?" >> gpurun_out/bench_r1h.err
for mb in resnet50:15 resnet50:16 resnet50:14 resnet50:32; do m=${mb%:*}; b=${mb#*:}
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_${m}_b$b.csv python tools/oneshot.py --model $m --batch $b --reps 3 > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/ncu_traffic_${m}_b$b.csv $m $b >> gpurun_out/oneshot_r1h.log 2>&1
done
cp profiles/ncu_*.json gpurun_out/ 2>/dev/null
timeout 120 python tools/oneshot.py --model resnet50 --batch 32 --json gpurun_out/trace_r1h_resnet50_b32.json >> gpurun_out/oneshot_r1h.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1h.csv python tools/oneshot.py --model resnet50 --batch 32 --reps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gl_executor -s 1 -c 1 -o gpurun_out/prof_r1h_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 2 > gpurun_out/ncufull_r1h.log 2>&1
echo done
