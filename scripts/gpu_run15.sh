mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi15.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests15.log 2>&1; echo "rc=$?" >> gpurun_out/gputests15.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.log 2>&1; echo "rc=$?" >> gpurun_out/smoke15.log
export GL_BENCH_WATCHDOG_S=500
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench15.json 2> gpurun_out/bench15.err; echo "rc=$?" >> gpurun_out/bench15.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches15_oneshot.csv python tools/oneshot.py --model resnet50 --batch 32 --reps 3 > gpurun_out/ncu15a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gl_executor -s 1 -c 1 -o gpurun_out/prof15_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 2 > gpurun_out/ncu15b.log 2>&1
