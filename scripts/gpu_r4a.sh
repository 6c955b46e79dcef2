# Round-2 first GPU pass: tests, smoke (plain + under ncu), profile re-measure on exact shares.
TAG=${1:-r4a}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches_$TAG.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_ncu_$TAG.log
timeout 900 python tools/profile_sweep.py --reps 10 --warmup 2 --out gpurun_out/profile_b200_$TAG.csv > gpurun_out/profile_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/profile_$TAG.log
