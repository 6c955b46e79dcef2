# Round-2 pass i: GPU suite + bench with the measured guard margin and the P:823 median criterion (2 runs).
TAG=${1:-r4i}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -o faulthandler_timeout=300 > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
timeout 1200 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --headline-only --margin 0 > gpurun_out/bench_${TAG}_m0.json 2> gpurun_out/bench_${TAG}_m0.log; echo "rc=$?" >> gpurun_out/bench_${TAG}_m0.log
