# Round-2: re-measure L(b, p) as the p90 host-observed service latency (R18), keep the
# ncu L2/DRAM features, then the bench on that profile (twice).
TAG=${1:-r5i}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
cp profiles/profile_b200.csv gpurun_out/profile_b200_median_$TAG.csv
timeout 900 python tools/profile_sweep.py --keep-stats profiles/profile_b200.csv --out gpurun_out/profile_b200_p90_$TAG.csv > gpurun_out/profile_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/profile_$TAG.log
cp gpurun_out/profile_b200_p90_$TAG.csv profiles/profile_b200.csv
timeout 1200 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --headline-only > gpurun_out/bench_${TAG}_rep2.json 2> gpurun_out/bench_${TAG}_rep2.log
