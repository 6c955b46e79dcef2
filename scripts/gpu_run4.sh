mkdir -p gpurun_out profiles
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for m in resnet50 vgg16 bert_base googlenet ssd_mobilenet_v1 lenet5; do
  timeout 300 python tools/oneshot.py --model $m --batch 32 --json gpurun_out/trace_${m}_b32.json >> gpurun_out/oneshot.log 2>&1
done
timeout 1500 python tools/profile_sweep.py --out gpurun_out/profile_b200.csv --reps 10 --warmup 2 > gpurun_out/profile.log 2>&1; echo "profile rc=$?" >> gpurun_out/profile.log
cp gpurun_out/profile_b200.csv profiles/profile_b200.csv
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
