# Round-2 experiment recipes (run under gpurun; results under profiles/):
#   bash scripts/ab_round2.sh tma-warps    # 1 vs 2 TMA-producer warps (profiles/ab_r4n_tma_producer_warps.log)
#   bash scripts/ab_round2.sh anatomy      # ResNet-50 b32 per-step anatomy under executor debug flags
#   bash scripts/ab_round2.sh gemm         # per-op GEMM tile timelines, BN x split-K sweeps
#   bash scripts/ab_round2.sh micro        # TMA / UMMA issue-rate microbenchmarks
#   bash scripts/ab_round2.sh kpair        # 1 vs 2 K blocks per ring stage (profiles/ab_r9a_kpair.log)
#   bash scripts/ab_round2.sh kpair2       # 2 / 4 K blocks per stage, >= 2 / 3 stages (profiles/ab_r9b_kpair2.log)
#   bash scripts/ab_round2.sh kpair-tw     # 1 vs 2 TMA-producer warps with paired stages (profiles/ab_r9c_kpair_tw.log)
# Variant libraries are built from the working tree with compile-time switches
# (GL_TMA_WARPS, GL_DBG_START) into paper_2109_01611_b200/_ab/ and passed as GL_LIB.
set -e
WHAT=${1:-tma-warps}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out paper_2109_01611_b200/_ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null
C=paper_2109_01611_b200
variant() {   # variant NAME FLAGS...: executor + runtime rebuilt with FLAGS, the rest reused
  local name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC "$@" -c $C/csrc/executor.cu -o /tmp/ex_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC "$@" -c $C/csrc/runtime.cpp -o /tmp/rt_$name.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $C/_ab/lib$name.so /tmp/ex_$name.o /tmp/rt_$name.o \
    $C/_build/detect.cu.o $C/_build/probe.cu.o $C/_build/models.cpp.o $C/_build/frontend.cpp.o \
    $C/_build/sched.cpp.o $C/_build/workload.cpp.o -lpthread -ldl -lrt
}
case $WHAT in
  tma-warps)
    variant tw1 -DGL_TMA_WARPS=1; variant tw2 -DGL_TMA_WARPS=2
    VARIANTS="tw1=$C/_ab/libtw1.so tw2=$C/_ab/libtw2.so" bash scripts/ab_oneshot.sh tmawarps \
      resnet50:1 resnet50:8 resnet50:32 bert_base:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:8 lenet5:32 ;;
  anatomy)
    for f in 0 2 1 4 8; do
      python tools/oneshot.py --model resnet50 --batch 32 --flags $f --json gpurun_out/trace_anatomy_f$f.json > /dev/null
    done
    variant dbgstart -DGL_DBG_START
    GL_LIB=$C/_ab/libdbgstart.so python tools/oneshot.py --model resnet50 --batch 1 --json gpurun_out/trace_dbgstart_b1.json ;;
  gemm)
    python tools/gemm_micro.py --only res_l4_3x3_512,res_l1_1x1_256,res_l1_3x3_64,res_l3_3x3_256 \
      --bn 0,64,128,256 --flags 0,8,4 --json gpurun_out/gemm_micro.json
    python tools/gemm_micro.py --only res_l4_3x3_512,res_l3_3x3_256,res_l2_3x3_128 --bn 64,128,256 \
      --split 1,2,4,8 --json gpurun_out/gemm_split.json ;;
  kpair)
    variant kp1 -DGL_KPAIR=1; variant kp2 -DGL_KPAIR=2
    VARIANTS="kp1=$C/_ab/libkp1.so kp2=$C/_ab/libkp2.so" bash scripts/ab_oneshot.sh kpair \
      resnet50:1 resnet50:8 resnet50:32 bert_base:8 bert_base:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:8 ;;
  kpair2)
    variant kp2m3 -DGL_KPAIR=2; variant kp2m2 -DGL_KPAIR=2 -DGL_KPAIR_MINST=2
    variant kp4m3 -DGL_KPAIR=4; variant kp4m2 -DGL_KPAIR=4 -DGL_KPAIR_MINST=2
    VARIANTS="kp2m3=$C/_ab/libkp2m3.so kp2m2=$C/_ab/libkp2m2.so kp4m3=$C/_ab/libkp4m3.so kp4m2=$C/_ab/libkp4m2.so" \
      bash scripts/ab_oneshot.sh kpair2 \
      resnet50:1 resnet50:8 resnet50:32 bert_base:8 bert_base:32 vgg16:32 googlenet:32 ssd_mobilenet_v1:8 ;;
  kpair-tw)
    variant kp2tw1 -DGL_TMA_WARPS=1; variant kp2tw2 -DGL_TMA_WARPS=2
    VARIANTS="kp2tw1=$C/_ab/libkp2tw1.so kp2tw2=$C/_ab/libkp2tw2.so" bash scripts/ab_oneshot.sh kpairtw \
      resnet50:1 resnet50:8 resnet50:32 bert_base:8 vgg16:32 googlenet:32 ssd_mobilenet_v1:8 ;;
  micro)
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I $C/csrc tools/tma_micro.cu -o tools/tma_micro -lcuda
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I $C/csrc tools/umma_micro.cu -o tools/umma_micro
    ./tools/tma_micro > gpurun_out/tma_micro.csv
    ./tools/umma_micro > gpurun_out/umma_micro.csv ;;
esac
