mkdir -p gpurun_out
timeout 600 python tools/gemm_micro.py --only res_l4_3x3_512,bert_ffn2,vgg_3x3_256_56 --flags 0,16,8,24,12,28 --json gpurun_out/micro22.json > gpurun_out/micro22.log 2>&1
timeout 300 python tools/profile_sweep.py --reps 10 --warmup 2 --out gpurun_out/profile_b200.csv > gpurun_out/profile22.log 2>&1
