mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests_r2s.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2s.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2s.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r2s.log
timeout 300 python tools/latency_ab.py > gpurun_out/lat_r2s.log 2>&1
export GL_BENCH_WATCHDOG_S=1400
timeout 1500 python bench.py --verbose > gpurun_out/bench_r2s.json 2> gpurun_out/bench_r2s.err; echo "rc=$?" >> gpurun_out/bench_r2s.err
echo done
