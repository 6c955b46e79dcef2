# Round-2 pass n: two TMA-producer warps (alternate K blocks) vs one (A/B), parity on the new build.
TAG=${1:-r4n}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
VARIANTS="tw1=paper_2109_01611_b200/_ab/libtw1.so tw2=paper_2109_01611_b200/_ab/libtw2.so" timeout 1500 bash scripts/ab_oneshot.sh ${TAG}tma resnet50:1 resnet50:8 resnet50:32 bert_base:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:8 lenet5:32 > gpurun_out/ab_${TAG}_tmawarps.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_models.py tests/test_gpu_fullsize.py tests/test_gpu_dataflow.py tests/test_gpu_executor.py tests/test_gpu_detect.py -m gpu -q > gpurun_out/gputests_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_$TAG.log
timeout 120 python tools/oneshot.py --model resnet50 --batch 32 --json gpurun_out/trace_${TAG}_resnet50_b32.json > /dev/null 2>&1
