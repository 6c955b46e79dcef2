mkdir -p gpurun_out
timeout 600 python tools/gemm_micro.py --only res_l1_1x1_64,res_l1_3x3_64,res_l3_3x3_256,vgg_3x3_256_56,bert_ffn1 --bn 0,128 --flags 0,1,2,4,8,12 --json gpurun_out/micro17.json > gpurun_out/micro17.log 2>&1
