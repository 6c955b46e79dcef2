# Tensor-pipe / TMA issue microbenchmarks (tools/umma_micro.cu, tools/tma_micro.cu).
TAG=${1:-r6}
mkdir -p gpurun_out
timeout 120 ./tools/umma_micro > gpurun_out/umma_micro_$TAG.csv 2>&1
timeout 120 ./tools/tma_micro > gpurun_out/tma_micro_$TAG.csv 2>&1
