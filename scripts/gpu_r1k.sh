mkdir -p gpurun_out
D=paper_2109_01611_b200/_ab
VARIANTS="A=$D/libgpulet_A.so Alds=$D/libgpulet_Alds.so Afin=$D/libgpulet_Afin.so B=paper_2109_01611_b200/libgpulet.so" bash scripts/ab_oneshot.sh k resnet50:32 resnet50:8 > gpurun_out/ab_k.log 2>&1
echo done
