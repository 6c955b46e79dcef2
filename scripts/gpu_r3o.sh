mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_r3o.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r3o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3o.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r3o.log
export GL_BENCH_WATCHDOG_S=600
for rep in 1 2; do timeout 700 python bench.py > gpurun_out/bench_r3o_rep$rep.json 2> gpurun_out/bench_r3o_rep$rep.err; done
echo done
