mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_serve.py -m gpu -q -x > gpurun_out/gputests_r1p.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1p.log
timeout 600 python tools/adapt.py --json gpurun_out/adapt_b200.json > gpurun_out/adapt_r1p.log 2>&1; echo "rc=$?" >> gpurun_out/adapt_r1p.log
export GL_BENCH_WATCHDOG_S=1100
timeout 1200 python bench.py --verbose > gpurun_out/bench_r1p.json 2> gpurun_out/bench_r1p.err; echo "rc=$?" >> gpurun_out/bench_r1p.err
echo done
