mkdir -p gpurun_out
export GL_BENCH_WATCHDOG_S=600
for rep in 1 2; do
  timeout 700 python bench.py > gpurun_out/bench_r3n_new_rep$rep.json 2> gpurun_out/bench_r3n_new_rep$rep.err
  GL_GUARD_MIN_US=5 GL_GUARD_DIV=20 timeout 700 python bench.py > gpurun_out/bench_r3n_old_rep$rep.json 2> gpurun_out/bench_r3n_old_rep$rep.err
done
echo done
