mkdir -p gpurun_out
timeout 600 python tools/gemm_micro.py --only res_l4_3x3_512,vgg_3x3_256_56,bert_ffn2,res_l1_3x3_64,res_conv1,res_l3_1x1_1024to256 --flags 0,1,2,4,8,12 --json gpurun_out/micro20.json > gpurun_out/micro20.log 2>&1
