# Round-2 closing pass on the final kernels (two K blocks per ring stage): smoke +
# its ncu launch list, the GPU parity suite, the p90 latency profile re-measured on
# these kernels, per-model one-shot traces, extras (floor, K12, cfg1), the per-point
# profile roofline, ncu DRAM traffic of the ResNet-50 lane's batches, one ncu --set
# full capture, the bench (full + headline repeat + reference arm), F1 / F3 / F4.
# Two parts (so the first results return early): PART=A smoke, tests, profile,
# traces, bench; PART=B extras, profile roofline, ncu traffic + full capture, F1/F3/F4.
TAG=${1:-r9}
PART=${2:-A}
mkdir -p gpurun_out
if [ "$PART" = A ]; then
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches_$TAG.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu_$TAG.log 2>&1
  timeout 1500 python -m pytest tests -m gpu -q -s -o faulthandler_timeout=300 > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
  timeout 1500 python tools/profile_sweep.py --keep-stats profiles/profile_b200.csv --out gpurun_out/profile_b200_$TAG.csv > gpurun_out/profile_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/profile_$TAG.log
  cp gpurun_out/profile_b200_$TAG.csv profiles/profile_b200.csv
  for mb in resnet50:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:32 bert_base:32 lenet5:32 resnet50:1; do m=${mb%:*}; b=${mb#*:}
    timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace_${TAG}_${m}_b${b}.json >> gpurun_out/oneshot_$TAG.log 2>&1
  done
  timeout 1500 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
  timeout 900 python bench.py --headline-only > gpurun_out/bench_${TAG}_rep2.json 2> gpurun_out/bench_${TAG}_rep2.log
  timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.log
else
  python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
  timeout 600 python tools/measure_extras.py --json gpurun_out/extras_$TAG.json > gpurun_out/extras_$TAG.log 2>&1
  timeout 400 python tools/profile_roofline.py --json gpurun_out/profile_roofline_$TAG.json > gpurun_out/profile_roofline_$TAG.log 2>&1
  for b in 24 26 28 30 32; do
    timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_resnet50_b$b.csv python tools/oneshot.py --model resnet50 --batch $b --reps 2 --n_sm 118 > /dev/null 2>&1
    python tools/ncu_traffic.py gpurun_out/ncu_traffic_resnet50_b$b.csv resnet50 $b >> gpurun_out/ncu_traffic_$TAG.log 2>&1
  done
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:gl_executor -c 1 -f -o gpurun_out/ncu_${TAG}_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
  timeout 900 python tools/adapt.py --json gpurun_out/adapt_$TAG.json > gpurun_out/adapt_$TAG.log 2>&1
  timeout 900 python tools/traffic_serve.py --json gpurun_out/traffic_serve_$TAG.json > gpurun_out/traffic_serve_$TAG.log 2>&1
  timeout 900 python tools/consolidate.py --secs 1.0 --json gpurun_out/consolidate_$TAG.json > gpurun_out/consolidate_$TAG.log 2>&1
fi
