# MMA-issuer loop shapes and TMA steady-state issue (tools/mma_loop_micro.cu, tools/tma_issue_micro.cu).
TAG=${1:-r6c}
mkdir -p gpurun_out
timeout 120 ./tools/mma_loop_micro > gpurun_out/mma_loop_micro_$TAG.csv 2>&1
timeout 120 ./tools/tma_issue_micro > gpurun_out/tma_issue_micro_$TAG.csv 2>&1
