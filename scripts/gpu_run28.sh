mkdir -p gpurun_out
timeout 600 python tools/gemm_micro.py --only res_l1_1x1_64,res_l1_1x1_256to64,res_l1_1x1_256,res_l1_3x3_64,res_conv1,vgg_3x3_256_56 --flags 0,1,2,12 --json gpurun_out/micro28.json > gpurun_out/micro28.log 2>&1
export GL_BENCH_WATCHDOG_S=600
timeout 700 python bench.py --verbose > gpurun_out/bench28.json 2> gpurun_out/bench28.err; echo "rc=$?" >> gpurun_out/bench28.err
