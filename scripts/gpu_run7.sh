mkdir -p gpurun_out
export GL_DEBUG=1
timeout 120 python -m pytest tests/test_gpu_executor.py -q -x -k "pair_confinement" > gpurun_out/exec7.log 2>&1; echo "exec rc=$?" >> gpurun_out/exec7.log
export GL_BENCH_WATCHDOG_S=150
timeout 200 python bench.py --steps 10 --warmup 3 --verbose --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "bench rc=$?" >> gpurun_out/bench7.err
