mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1i.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1i.log
for mb in resnet50:32 resnet50:8 bert_base:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:32 lenet5:24; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace_r1i_${m}_b${b}.json >> gpurun_out/oneshot_r1i.log 2>&1
done
export GL_BENCH_WATCHDOG_S=1100
timeout 1200 python bench.py --verbose > gpurun_out/bench_r1i.json 2> gpurun_out/bench_r1i.err; echo "rc=$?" >> gpurun_out/bench_r1i.err
echo done
