mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
VARIANTS="Alds=$D/libgpulet_Alds.so C1=$D/libgpulet_C1.so C2=$D/libgpulet_C2.so" bash scripts/ab_oneshot.sh l resnet50:32 resnet50:8 resnet50:15 bert_base:32 > gpurun_out/ab_l.log 2>&1
echo done
