# Round-2 pass c: new parity tests (top-1 over 256/1024 requests, BERT pooled vector,
# unconfined executors), ResNet-50 b32 per-step anatomy under executor debug flags,
# LeNet+VGG consolidation curves with the unconfined (MPS(default)) analogue.
TAG=${1:-r4c}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_top1.py tests/test_gpu_models.py tests/test_gpu_fullsize.py tests/test_gpu_executor.py tests/test_gpu_dataflow.py -m gpu -q -s > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
for f in 0 2 1 4 8; do
  timeout 120 python tools/oneshot.py --model resnet50 --batch 32 --flags $f --json gpurun_out/trace_${TAG}_resnet50_b32_f$f.json > gpurun_out/oneshot_${TAG}_f$f.log 2>&1
done
timeout 900 python tools/consolidate.py --secs 1.0 --json gpurun_out/consolidate_$TAG.json > gpurun_out/consolidate_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/consolidate_$TAG.log
timeout 300 python -m pytest tests/test_gpu_serve.py -m gpu -q > gpurun_out/gputests_serve_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_serve_$TAG.log
timeout 1200 python tools/traffic_serve.py --json gpurun_out/traffic_serve_$TAG.json > gpurun_out/traffic_serve_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/traffic_serve_$TAG.log
