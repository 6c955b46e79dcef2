# Round-2 pass p: three TMA-producer warps vs two (A/B).
TAG=${1:-r4p}
mkdir -p gpurun_out
VARIANTS="tw2=paper_2109_01611_b200/_ab/libtw2.so tw3=paper_2109_01611_b200/_ab/libtw3.so" timeout 1500 bash scripts/ab_oneshot.sh ${TAG}tma resnet50:1 resnet50:8 resnet50:32 bert_base:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:8 > gpurun_out/ab_${TAG}_tmawarps.log 2>&1
