# Round-2 pass j: gpu-let barrier with arrival counters spread over 8 lines vs one line (A/B), parity.
TAG=${1:-r4j}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
VARIANTS="one=paper_2109_01611_b200/_ab/libbar1.so spread=paper_2109_01611_b200/_ab/libbar8.so" timeout 1200 bash scripts/ab_oneshot.sh ${TAG}bar resnet50:1 resnet50:8 resnet50:32 bert_base:32 googlenet:8 ssd_mobilenet_v1:8 > gpurun_out/ab_${TAG}_barrier.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py tests/test_gpu_fullsize.py tests/test_gpu_dataflow.py tests/test_gpu_executor.py tests/test_gpu_serve.py -m gpu -q > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
