mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests_r1u.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1u.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r1u.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_r1u.log
timeout 600 python tools/adapt.py --json gpurun_out/adapt_b200.json > gpurun_out/adapt_r1u.log 2>&1; echo "rc=$?" >> gpurun_out/adapt_r1u.log
for b in 15 32; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1u_resnet50_b$b.csv python tools/oneshot.py --model resnet50 --batch $b --reps 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gl_executor -s 1 -c 1 -o gpurun_out/prof_r1u_resnet50_b$b python tools/oneshot.py --model resnet50 --batch $b --reps 2 > gpurun_out/ncufull_r1u_b$b.log 2>&1
done
timeout 120 python tools/oneshot.py --model resnet50 --batch 15 --json gpurun_out/trace_r1u_resnet50_b15.json > /dev/null 2>&1
echo done
