# Round-2 pass g: per-op GEMM anatomy (tile timelines) of ResNet-50 b32 shapes under BN / debug-flag sweeps.
TAG=${1:-r4g}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python tools/gemm_micro.py --only res_l4_3x3_512,res_l1_1x1_256,res_l1_3x3_64,res_l3_3x3_256,res_l3_1x1_256to1024 --bn 0,64,128,256 --flags 0,8,4 --json gpurun_out/gemm_micro_$TAG.json > gpurun_out/gemm_micro_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_micro_$TAG.log
