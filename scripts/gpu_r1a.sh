# Round-1 re-entry measurement: GPU tests, smoke, bench, ncu launch list + full capture.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_r1a.txt 2>&1
cat MEASURED_PEAKS.json > gpurun_out/peaks_r1a.json 2>/dev/null
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1a.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1a.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r1a.log
export GL_BENCH_WATCHDOG_S=900
timeout 1000 python bench.py --verbose > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; echo "rc=$?" >> gpurun_out/bench_r1a.err
for mb in resnet50:32 resnet50:8 vgg16:32 bert_base:32 lenet5:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace_r1a_${m}_b${b}.json >> gpurun_out/oneshot_r1a.log 2>&1
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_${m}_b$b.csv python tools/oneshot.py --model $m --batch $b --reps 3 > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/ncu_traffic_${m}_b$b.csv $m $b >> gpurun_out/oneshot_r1a.log 2>&1
done
cp profiles/ncu_*.json gpurun_out/ 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv python tools/oneshot.py --model resnet50 --batch 32 --reps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gl_executor -s 1 -c 1 -o gpurun_out/prof_r1a_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 2 > gpurun_out/ncufull_r1a.log 2>&1
echo done
