mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests_r1y.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1y.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1y.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r1y.log
timeout 600 python tools/adapt.py --scenario traffic --json gpurun_out/adapt_traffic_b200.json > gpurun_out/adapt_traffic_r1y.log 2>&1; echo "rc=$?" >> gpurun_out/adapt_traffic_r1y.log
export GL_BENCH_WATCHDOG_S=1400
timeout 1500 python bench.py --verbose > gpurun_out/bench_r1y.json 2> gpurun_out/bench_r1y.err; echo "rc=$?" >> gpurun_out/bench_r1y.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r1y.json 2> gpurun_out/bench_ref_r1y.err; echo "rc=$?" >> gpurun_out/bench_ref_r1y.err
echo done
