mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_r2z.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r2z.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2z.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r2z.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2z_resnet50_b15.csv python tools/oneshot.py --model resnet50 --batch 15 --reps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gl_executor -s 1 -c 1 -o gpurun_out/prof_r2z_resnet50_b15 python tools/oneshot.py --model resnet50 --batch 15 --reps 2 > gpurun_out/ncufull_r2z.log 2>&1
echo done
