# Round-2 pass d: residual-TMA epilogue parity + A/B, chain-serve hang diagnosis,
# LeNet guard-margin diagnostic, extras, consolidation and traffic chain serving.
TAG=${1:-r4d}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 200 python -m pytest tests/test_gpu_serve.py -k chain -q -s -o faulthandler_timeout=60 > gpurun_out/chain_dbg_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/chain_dbg_$TAG.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py tests/test_gpu_fullsize.py tests/test_gpu_top1.py tests/test_gpu_dataflow.py -m gpu -q -s > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
VARIANTS="base=paper_2109_01611_b200/_ab/libbase.so rtma=paper_2109_01611_b200/_ab/librtma.so" timeout 900 bash scripts/ab_oneshot.sh ${TAG}rtma resnet50:32 resnet50:15 resnet50:8 bert_base:32 > gpurun_out/ab_${TAG}_rtma.log 2>&1
timeout 120 python tools/oneshot.py --model resnet50 --batch 32 --json gpurun_out/trace_${TAG}_resnet50_b32.json > /dev/null 2>&1
timeout 600 python scripts/diag_margin.py 1.0,2.5 gpurun_out/diag_margin_$TAG.json > gpurun_out/diag_margin_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/diag_margin_$TAG.log
timeout 300 python tools/measure_extras.py --json gpurun_out/extras_$TAG.json > gpurun_out/extras_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/extras_$TAG.log
timeout 900 python tools/consolidate.py --secs 1.0 --json gpurun_out/consolidate_$TAG.json > gpurun_out/consolidate_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/consolidate_$TAG.log
timeout 900 python tools/traffic_serve.py --json gpurun_out/traffic_serve_$TAG.json > gpurun_out/traffic_serve_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/traffic_serve_$TAG.log
