mkdir -p gpurun_out
export GL_BENCH_WATCHDOG_S=600
for rep in 1 2 3; do timeout 700 python bench.py > gpurun_out/bench_r3k_rep$rep.json 2> gpurun_out/bench_r3k_rep$rep.err; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r3k.json 2> gpurun_out/bench_ref_r3k.err
echo done
