mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_serve.py tests/test_gpu_executor.py -m gpu -q > gpurun_out/gputests_r2u.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2u.log
export GL_BENCH_WATCHDOG_S=1400
timeout 1500 python bench.py --verbose --headline-only > gpurun_out/bench_r2u.json 2> gpurun_out/bench_r2u.err; echo "rc=$?" >> gpurun_out/bench_r2u.err
echo done
