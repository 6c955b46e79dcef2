mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_detect.py -q -x > gpurun_out/gputests_r3e_detect.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r3e_detect.log
timeout 300 python tools/traffic_pipeline.py --batch 8 --per-img 4 --json gpurun_out/traffic_pipeline_b200.json > gpurun_out/pipeline_r3e.log 2>&1; echo "rc=$?" >> gpurun_out/pipeline_r3e.log
timeout 300 python tools/traffic_pipeline.py --batch 8 --per-img 4 --score-thr 0.2 --json gpurun_out/traffic_pipeline_thr02_b200.json >> gpurun_out/pipeline_r3e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssd_ -c 2 -o gpurun_out/prof_r3e_detect python tools/traffic_pipeline.py --reps 1 > gpurun_out/ncu_r3e.log 2>&1
echo done
