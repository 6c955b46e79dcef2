mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_detect.py -q -x > gpurun_out/gputests_r3d_detect.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r3d_detect.log
timeout 300 python tools/traffic_pipeline.py --batch 8 --per-img 4 --json gpurun_out/traffic_pipeline_b200.json > gpurun_out/pipeline_r3d.log 2>&1; echo "rc=$?" >> gpurun_out/pipeline_r3d.log
timeout 300 python tools/traffic_pipeline.py --batch 4 --per-img 2 --score-thr 0.05 --json gpurun_out/traffic_pipeline_b4_b200.json >> gpurun_out/pipeline_r3d.log 2>&1; echo "rc=$?" >> gpurun_out/pipeline_r3d.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r3d_pipeline.csv python tools/traffic_pipeline.py --reps 2 > /dev/null 2>&1
echo done
