mkdir -p gpurun_out
export GL_BENCH_WATCHDOG_S=300
timeout 400 python bench.py --steps 5 --warmup 2 --verbose --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc=$?" >> gpurun_out/bench5.err
timeout 300 python tools/oneshot.py --model resnet50 --batch 1 --json gpurun_out/trace_resnet50_b1.json > gpurun_out/oneshot_b1.log 2>&1
timeout 300 python tools/oneshot.py --model bert_base --batch 1 --json gpurun_out/trace_bert_base_b1.json >> gpurun_out/oneshot_b1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gl_executor -s 1 -c 1 -o gpurun_out/ncu_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 2 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gl_executor -s 1 -c 1 -o gpurun_out/ncu_resnet50_b1 python tools/oneshot.py --model resnet50 --batch 1 --reps 2 > gpurun_out/ncu2.log 2>&1
