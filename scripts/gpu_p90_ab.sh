# Same-box A/B of the latency-profile statistic (R18): the committed median profile
# vs a freshly measured p90-of-50 profile, headline-only bench runs interleaved,
# then the periodic-rescheduling trace (F1) on the committed profile.
TAG=${1:-r6p}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
cp profiles/profile_b200.csv gpurun_out/profile_b200_median_$TAG.csv
timeout 900 python bench.py --headline-only --no-cpu-baseline > gpurun_out/bench_${TAG}_med1.json 2> gpurun_out/bench_${TAG}_med1.log
timeout 1500 python tools/profile_sweep.py --keep-stats profiles/profile_b200.csv --out gpurun_out/profile_b200_p90_$TAG.csv > gpurun_out/profile_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/profile_$TAG.log
cp gpurun_out/profile_b200_p90_$TAG.csv profiles/profile_b200.csv
timeout 900 python bench.py --headline-only --no-cpu-baseline > gpurun_out/bench_${TAG}_p90a.json 2> gpurun_out/bench_${TAG}_p90a.log
cp gpurun_out/profile_b200_median_$TAG.csv profiles/profile_b200.csv
timeout 900 python bench.py --headline-only --no-cpu-baseline > gpurun_out/bench_${TAG}_med2.json 2> gpurun_out/bench_${TAG}_med2.log
cp gpurun_out/profile_b200_p90_$TAG.csv profiles/profile_b200.csv
timeout 900 python bench.py --headline-only --no-cpu-baseline > gpurun_out/bench_${TAG}_p90b.json 2> gpurun_out/bench_${TAG}_p90b.log
cp gpurun_out/profile_b200_median_$TAG.csv profiles/profile_b200.csv
timeout 900 python tools/adapt.py --json gpurun_out/adapt_$TAG.json > gpurun_out/adapt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/adapt_$TAG.log
