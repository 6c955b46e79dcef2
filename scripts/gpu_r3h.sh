mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_r3h.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r3h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r3h.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r3h.log
timeout 300 python tools/traffic_pipeline.py --batch 8 --per-img 4 --json gpurun_out/traffic_pipeline_b200.json > gpurun_out/pipeline_r3h.log 2>&1; echo "rc=$?" >> gpurun_out/pipeline_r3h.log
timeout 300 python tools/traffic_pipeline.py --batch 8 --per-img 4 --score-thr 0.2 --json gpurun_out/traffic_pipeline_thr02_b200.json >> gpurun_out/pipeline_r3h.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r3h_pipeline.csv python tools/traffic_pipeline.py --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssd_ -c 2 -o gpurun_out/prof_r3h_detect python tools/traffic_pipeline.py --reps 1 > gpurun_out/ncu_r3h.log 2>&1
echo done
