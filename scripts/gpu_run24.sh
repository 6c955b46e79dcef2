mkdir -p gpurun_out
timeout 600 python tools/profile_sweep.py --reps 10 --warmup 2 > gpurun_out/profile24.log 2>&1; echo "rc=$?" >> gpurun_out/profile24.log
cp profiles/profile_b200.csv gpurun_out/profile_b200_lat.csv
timeout 900 ncu --metrics lts__t_sectors.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum -k regex:gl_executor --csv --log-file gpurun_out/ncu_stats24.csv python tools/ncu_stats.py launch > gpurun_out/ncu24.log 2>&1; echo "rc=$?" >> gpurun_out/ncu24.log
python tools/ncu_stats.py apply gpurun_out/ncu_stats24.csv >> gpurun_out/ncu24.log 2>&1
cp profiles/profile_b200.csv gpurun_out/profile_b200.csv
timeout 900 python tools/corun.py --batches 2,8,32 --splits 20,50,80 --ms 120 > gpurun_out/corun24.log 2>&1; echo "rc=$?" >> gpurun_out/corun24.log
cp profiles/coeffs_b200.json profiles/corun_b200.csv gpurun_out/ 2>/dev/null
export GL_BENCH_WATCHDOG_S=600
timeout 700 python bench.py --verbose > gpurun_out/bench24.json 2> gpurun_out/bench24.err; echo "rc=$?" >> gpurun_out/bench24.err
