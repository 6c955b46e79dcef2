# Same-box A/B of the latency-profile statistic (R18), round-2 closing kernels:
# p90 of 50 (the committed reading) vs p99 of 200 host-observed service latencies,
# both measured on this box, headline-only bench runs interleaved; then one ncu
# --set full capture of a ResNet-50 b32 launch.
TAG=${1:-r9p}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
cp profiles/profile_b200.csv /tmp/keep_stats.csv
timeout 900 python tools/profile_sweep.py --keep-stats /tmp/keep_stats.csv --out gpurun_out/profile_b200_p90_$TAG.csv > gpurun_out/profile_p90_$TAG.log 2>&1
timeout 1500 python tools/profile_sweep.py --keep-stats /tmp/keep_stats.csv --reps 200 --quantile 0.99 --out gpurun_out/profile_b200_p99_$TAG.csv > gpurun_out/profile_p99_$TAG.log 2>&1
for run in p90a p99a p90b p99b; do
  cp gpurun_out/profile_b200_${run%?}_$TAG.csv profiles/profile_b200.csv
  timeout 900 python bench.py --headline-only --no-cpu-baseline > gpurun_out/bench_${TAG}_$run.json 2> gpurun_out/bench_${TAG}_$run.log
done
cp /tmp/keep_stats.csv profiles/profile_b200.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gl_executor -c 1 -f -o gpurun_out/ncu_${TAG}_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
