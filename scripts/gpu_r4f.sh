# Round-2 pass f: full GPU suite + smoke, extras (publish probe), bench (8 retries, per-window violations).
TAG=${1:-r4f}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -o faulthandler_timeout=300 > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
timeout 400 python tools/measure_extras.py --json gpurun_out/extras_$TAG.json > gpurun_out/extras_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/extras_$TAG.log
timeout 1200 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
