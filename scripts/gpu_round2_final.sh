# Round-2 final measurement pass on one B200 (run under gpurun): full GPU suite and
# smoke, the whole measurement pipeline on the final executor (profile, ncu L2/DRAM
# stats, co-runs + fit, K12/floor/cfg1/publish extras, traces), per-point profile
# roofline, ncu DRAM traffic of the ResNet-50 lane's batches on its 118-SM share,
# one ncu --set full capture + launch list, consolidation (F4), traffic chain (F3),
# periodic rescheduling (F1), and the bench (ours x2, reference).
TAG=${1:-r5}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -s -o faulthandler_timeout=300 > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches_$TAG.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_ncu_$TAG.log 2>&1
bash scripts/measure_all.sh $TAG
cp gpurun_out/profile_b200.csv gpurun_out/coeffs_b200.json gpurun_out/corun_b200.csv profiles/ 2>/dev/null
cp gpurun_out/extras_$TAG.json profiles/extras_b200.json 2>/dev/null
timeout 400 python tools/profile_roofline.py --json gpurun_out/profile_roofline_$TAG.json > gpurun_out/profile_roofline_$TAG.log 2>&1
for b in 16 18 20 22 24 26 27 28 30 32; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_resnet50_b$b.csv python tools/oneshot.py --model resnet50 --batch $b --reps 2 --n_sm 118 > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/ncu_traffic_resnet50_b$b.csv resnet50 $b >> gpurun_out/ncu_traffic_$TAG.log 2>&1
done
cp profiles/ncu_resnet50_b*.json gpurun_out/ 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gl_executor -c 1 -f -o gpurun_out/ncu_${TAG}_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 python tools/consolidate.py --secs 1.0 --json gpurun_out/consolidate_$TAG.json > gpurun_out/consolidate_$TAG.log 2>&1
timeout 900 python tools/traffic_serve.py --json gpurun_out/traffic_serve_$TAG.json > gpurun_out/traffic_serve_$TAG.log 2>&1
timeout 900 python tools/adapt.py --json gpurun_out/adapt_$TAG.json > gpurun_out/adapt_$TAG.log 2>&1
timeout 1200 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
timeout 900 python bench.py --headline-only > gpurun_out/bench_${TAG}_rep2.json 2> gpurun_out/bench_${TAG}_rep2.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.log
