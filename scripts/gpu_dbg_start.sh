# Step-start anatomy with the GL_DBG_START build (abl/libD.so): CTA 0's stamps per
# GEMM step: [2] step entry, [4] args staged, [5] producer before the proxy fence,
# [0] after it (first TMA), relative to the previous barrier's release.
mkdir -p gpurun_out
for mb in resnet50:8 resnet50:32 resnet50:1; do m=${mb%:*}; b=${mb#*:}
  GL_LIB=abl/libD.so timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --json gpurun_out/dbgstart_${m}_b${b}.json > /dev/null 2>&1
done
