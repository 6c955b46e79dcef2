mkdir -p gpurun_out
timeout 600 python tools/adapt.py --json gpurun_out/adapt_b200.json > gpurun_out/adapt_r1q.log 2>&1; echo "rc=$?" >> gpurun_out/adapt_r1q.log
export GL_BENCH_WATCHDOG_S=1400
timeout 1500 python bench.py --verbose > gpurun_out/bench_r1q.json 2> gpurun_out/bench_r1q.err; echo "rc=$?" >> gpurun_out/bench_r1q.err
echo done
