mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/exec10.log 2>&1; echo "exec rc=$?" >> gpurun_out/exec10.log
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kern10.log 2>&1; echo "kern rc=$?" >> gpurun_out/kern10.log
timeout 300 python -m pytest tests/test_gpu_models.py -q -x > gpurun_out/models10.log 2>&1; echo "models rc=$?" >> gpurun_out/models10.log
for mb in resnet50:1 resnet50:32 vgg16:32 bert_base:32 googlenet:32 ssd_mobilenet_v1:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace10_${m}_b${b}.json >> gpurun_out/oneshot10.log 2>&1
done
export GL_BENCH_WATCHDOG_S=250
timeout 300 python bench.py --steps 10 --warmup 3 --verbose --no-cpu-baseline > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo "bench rc=$?" >> gpurun_out/bench10.err
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gl_executor -s 1 -c 1 -o gpurun_out/ncu10_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 2 > gpurun_out/ncu10.log 2>&1
