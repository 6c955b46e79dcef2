# Quick GPU validation pass: build, smoke, GPU parity suite, one bench line.
TAG=${1:-r6a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -s -o faulthandler_timeout=300 > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
