# Issue-rate microbenchmarks with loop-invariant operands (tools/umma_issue_micro.cu, tools/tma_issue_micro.cu).
TAG=${1:-r6b}
mkdir -p gpurun_out
timeout 120 ./tools/umma_issue_micro > gpurun_out/umma_issue_micro_$TAG.csv 2>&1
timeout 120 ./tools/tma_issue_micro > gpurun_out/tma_issue_micro_$TAG.csv 2>&1
