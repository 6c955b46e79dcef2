mkdir -p gpurun_out
export GL_DEBUG=1
timeout 240 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/exec8.log 2>&1; echo "exec rc=$?" >> gpurun_out/exec8.log
unset GL_DEBUG
timeout 300 python -m pytest tests/test_gpu_models.py -q -x > gpurun_out/models8.log 2>&1; echo "models rc=$?" >> gpurun_out/models8.log
export GL_BENCH_WATCHDOG_S=250
timeout 300 python bench.py --steps 10 --warmup 3 --verbose > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo "bench rc=$?" >> gpurun_out/bench8.err
for mb in resnet50:1 resnet50:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace8_${m}_b${b}.json >> gpurun_out/oneshot8.log 2>&1
done
