mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests23.log 2>&1; echo "rc=$?" >> gpurun_out/gputests23.log
for mb in resnet50:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace23_${m}_b${b}.json >> gpurun_out/oneshot23.log 2>&1
done
export GL_BENCH_WATCHDOG_S=500
timeout 600 python bench.py --verbose > gpurun_out/bench23.json 2> gpurun_out/bench23.err; echo "rc=$?" >> gpurun_out/bench23.err
