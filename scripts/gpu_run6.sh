mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/kern6.log 2>&1; echo "kern rc=$?" >> gpurun_out/kern6.log
timeout 600 python -m pytest tests/test_gpu_executor.py tests/test_gpu_models.py -q -x > gpurun_out/models6.log 2>&1; echo "models rc=$?" >> gpurun_out/models6.log
for mb in resnet50:1 resnet50:32 bert_base:32 vgg16:32 lenet5:32; do m=${mb%:*}; b=${mb#*:}
  timeout 300 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace6_${m}_b${b}.json >> gpurun_out/oneshot6.log 2>&1
done
export GL_BENCH_WATCHDOG_S=400
timeout 500 python bench.py --steps 10 --warmup 3 --verbose > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo "bench rc=$?" >> gpurun_out/bench6.err
