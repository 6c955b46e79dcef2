mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_detect.py -q -x > gpurun_out/gputests_r3j_detect.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r3j_detect.log
timeout 300 python tools/traffic_pipeline.py --batch 8 --per-img 4 --json gpurun_out/traffic_pipeline_b200.json > gpurun_out/pipeline_r3j.log 2>&1; echo "rc=$?" >> gpurun_out/pipeline_r3j.log
timeout 300 python tools/traffic_pipeline.py --batch 8 --per-img 4 --score-thr 0.2 --json gpurun_out/traffic_pipeline_thr02_b200.json >> gpurun_out/pipeline_r3j.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r3j_pipeline.csv python tools/traffic_pipeline.py --reps 2 > /dev/null 2>&1
echo done
