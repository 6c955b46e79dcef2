# Full measurement pipeline on one B200 (run under gpurun): latency profile
# L(b,p), ncu L2/DRAM stats, co-run interference fit, K12 probe + executor
# floor + cfg1, per-model traces.  Results under gpurun_out/ (copy the ones to
# keep into profiles/).
TAG=${1:-run}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 600 python tools/profile_sweep.py --reps 10 --warmup 2 > gpurun_out/profile_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/profile_$TAG.log
timeout 1200 ncu --metrics lts__t_sectors.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum -k regex:gl_executor --csv --log-file gpurun_out/ncu_stats_$TAG.csv python tools/ncu_stats.py launch > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_stats.py apply gpurun_out/ncu_stats_$TAG.csv >> gpurun_out/ncu_$TAG.log 2>&1
timeout 1800 python tools/corun.py --models lenet5,googlenet,resnet50,ssd_mobilenet_v1,vgg16,bert_base --batches ${CORUN_B:-2,4,8,16,32} --splits ${CORUN_S:-20,40,50,60,80} --ms ${CORUN_MS:-200} > gpurun_out/corun_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/corun_$TAG.log
cp profiles/profile_b200.csv profiles/coeffs_b200.json profiles/corun_b200.csv gpurun_out/ 2>/dev/null
timeout 600 python tools/measure_extras.py --json gpurun_out/extras_$TAG.json > gpurun_out/extras_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/extras_$TAG.log
for mb in resnet50:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:32 bert_base:32 lenet5:32 resnet50:1; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --json gpurun_out/trace_${TAG}_${m}_b${b}.json >> gpurun_out/oneshot_$TAG.log 2>&1
done
