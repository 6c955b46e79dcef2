mkdir -p gpurun_out
export GL_BENCH_WATCHDOG_S=1400
for r in 1 2 3; do
timeout 900 python bench.py --headline-only --no-e2e --no-cpu-baseline > gpurun_out/bench_rep_$r.json 2> gpurun_out/bench_rep_$r.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2y.json 2>&1
echo done
