mkdir -p gpurun_out
timeout 900 python tools/consolidate.py --json gpurun_out/consolidate_b200.json > gpurun_out/consolidate_r3c.log 2>&1; echo "rc=$?" >> gpurun_out/consolidate_r3c.log
timeout 900 python tools/adapt.py --json gpurun_out/adapt_b200.json > gpurun_out/adapt_r3c.log 2>&1; echo "rc=$?" >> gpurun_out/adapt_r3c.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r3c_lenet5_b32.csv python tools/oneshot.py --model lenet5 --batch 32 --reps 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gl_executor -s 1 -c 1 -o gpurun_out/prof_r3c_lenet5_b32 python tools/oneshot.py --model lenet5 --batch 32 --reps 2 > gpurun_out/ncufull_r3c.log 2>&1
export GL_BENCH_WATCHDOG_S=600
for rep in 1 2; do timeout 700 python bench.py > gpurun_out/bench_r3c_rep$rep.json 2> gpurun_out/bench_r3c_rep$rep.err; done
echo done
