# Round-2 closing measurement on one B200 with the p90 profile (R18): smoke + its
# ncu launch list, the GPU parity suite, the bench (full with the scenario x mode
# matrix, a headline repeat, the reference arm), periodic rescheduling (F1), the
# traffic chain (F3) and the consolidation curves (F4).
TAG=${1:-r6z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches_$TAG.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_ncu_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -s -o faulthandler_timeout=300 > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
timeout 1500 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --headline-only > gpurun_out/bench_${TAG}_rep2.json 2> gpurun_out/bench_${TAG}_rep2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.log
timeout 900 python tools/adapt.py --json gpurun_out/adapt_$TAG.json > gpurun_out/adapt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/adapt_$TAG.log
timeout 900 python tools/traffic_serve.py --json gpurun_out/traffic_serve_$TAG.json > gpurun_out/traffic_serve_$TAG.log 2>&1
timeout 900 python tools/consolidate.py --secs 1.0 --json gpurun_out/consolidate_$TAG.json > gpurun_out/consolidate_$TAG.log 2>&1
