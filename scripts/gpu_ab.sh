# Correctness of the working-tree library (GEMM kernels + models) then an interleaved
# one-shot A/B of the libraries in abl/ (VARIANTS="A=abl/libA.so B=abl/libB.so" by default).
#   bash scripts/gpu_ab.sh TAG [model:batch ...]
TAG=$1; shift 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py -m gpu -x -q > gpurun_out/ab_${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_${TAG}_tests.log
VARIANTS=${VARIANTS:-"A=abl/libA.so B=abl/libB.so"} bash scripts/ab_oneshot.sh $TAG "$@" > gpurun_out/ab_${TAG}.log 2>&1
