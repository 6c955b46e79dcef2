# Round-2 pass h: BN x split-K sweep of the A-shared small-M convolutions (L2 hot-spot hypothesis).
TAG=${1:-r4h}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python tools/gemm_micro.py --only res_l4_3x3_512,res_l3_3x3_256,res_l2_3x3_128,res_l3_1x1_1024to256 --bn 64,128,256 --split 1,2,4,8 --json gpurun_out/gemm_split_$TAG.json > gpurun_out/gemm_split_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_split_$TAG.log
