mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1e.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1e.log
for fl in 0 32; do for mb in resnet50:32 resnet50:8 bert_base:32; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --flags $fl --json gpurun_out/trace_r1e_f${fl}_${m}_b${b}.json >> gpurun_out/oneshot_r1e.log 2>&1
done; done
timeout 600 python tools/gemm_micro.py --only res_l1_1x1_64,res_l1_1x1_256,res_l3_3x3_256 --flags 0,32 --json gpurun_out/micro_r1e.json > gpurun_out/micro_r1e.log 2>&1
export GL_BENCH_WATCHDOG_S=900
timeout 900 python bench.py --verbose --headline-only --steps 4 --warmup 3 > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err; echo "rc=$?" >> gpurun_out/bench_r1e.err
echo done
