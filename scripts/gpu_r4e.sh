# Round-2 pass e: chain-serve test, ms-stall diagnosis, ncu source capture of the
# ResNet-50 b32 executor launch, extras (cfg1), per-point profile roofline, bench.
TAG=${1:-r4e}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 300 python -m pytest tests/test_gpu_serve.py -q -s -o faulthandler_timeout=120 > gpurun_out/gputests_serve_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_serve_$TAG.log
timeout 400 python scripts/diag_stall.py gpurun_out/diag_stall_$TAG.json > gpurun_out/diag_stall_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/diag_stall_$TAG.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gl_executor -c 1 -f -o gpurun_out/ncu_${TAG}_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_$TAG.log
timeout 400 python tools/measure_extras.py --json gpurun_out/extras_$TAG.json > gpurun_out/extras_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/extras_$TAG.log
timeout 400 python tools/profile_roofline.py --json gpurun_out/profile_roofline_$TAG.json > gpurun_out/profile_roofline_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/profile_roofline_$TAG.log
timeout 900 python bench.py --verbose > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.log; echo "rc=$?" >> gpurun_out/bench_$TAG.log
