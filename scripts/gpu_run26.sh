mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests26.log 2>&1; echo "rc=$?" >> gpurun_out/gputests25.log
timeout 600 python tools/gemm_micro.py --json gpurun_out/micro26.json > gpurun_out/micro26.log 2>&1
for mb in resnet50:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:32 bert_base:32 lenet5:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace26_${m}_b${b}.json >> gpurun_out/oneshot26.log 2>&1
done
for b in 16 24 32; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_resnet50_b$b.csv python tools/oneshot.py --model resnet50 --batch $b --reps 3 > /dev/null 2>&1
  python tools/ncu_traffic.py gpurun_out/ncu_traffic_resnet50_b$b.csv resnet50 $b >> gpurun_out/oneshot26.log 2>&1
done
cp profiles/ncu_*.json gpurun_out/ 2>/dev/null
export GL_BENCH_WATCHDOG_S=600
timeout 700 python bench.py --verbose > gpurun_out/bench26.json 2> gpurun_out/bench26.err; echo "rc=$?" >> gpurun_out/bench26.err
