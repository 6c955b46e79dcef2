# Round-2 bench repeat: default bench (measured p99.9 guard margins), headline with margin 0, F1 adapt.
TAG=${1:-r5b}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1200 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --headline-only --margin 0 > gpurun_out/bench_${TAG}_m0.json 2> gpurun_out/bench_${TAG}_m0.log
timeout 900 python tools/adapt.py --json gpurun_out/adapt_$TAG.json > gpurun_out/adapt_$TAG.log 2>&1
