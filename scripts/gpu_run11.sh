mkdir -p gpurun_out
timeout 100 python scripts/diag_pairs.py > gpurun_out/diag_a.log 2>&1
GL_SLOT1_FORWARD=9 timeout 100 python scripts/diag_pairs.py > gpurun_out/diag_b.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gl_executor -s 1 -c 1 -o gpurun_out/ncu11_resnet50_b32 python tools/oneshot.py --model resnet50 --batch 32 --reps 2 > gpurun_out/ncu11.log 2>&1
