mkdir -p gpurun_out
for pq in "50 50" "20 80" "80 20" "60 40" "40 60"; do timeout 60 python scripts/diag_pairs.py $pq >> gpurun_out/diag14.log 2>&1; done
timeout 200 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/exec14.log 2>&1; echo "exec rc=$?" >> gpurun_out/exec14.log
timeout 900 python tools/profile_sweep.py --out gpurun_out/profile_b200.csv --reps 10 --warmup 2 > gpurun_out/profile14.log 2>&1; echo "profile rc=$?" >> gpurun_out/profile14.log
cp gpurun_out/profile_b200.csv profiles/profile_b200.csv
export GL_BENCH_WATCHDOG_S=250
timeout 300 python bench.py --steps 10 --warmup 3 --verbose --no-cpu-baseline > gpurun_out/bench14.json 2> gpurun_out/bench14.err; echo "bench rc=$?" >> gpurun_out/bench14.err
