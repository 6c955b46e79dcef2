mkdir -p gpurun_out
for r in 1 2; do
timeout 300 python tools/serve_ab.py --xs 2.27,2.5 > gpurun_out/ab_g_new_$r.log 2>&1
GL_LIB=paper_2109_01611_b200/_ab/libgpulet_nopf.so timeout 300 python tools/serve_ab.py --xs 2.27,2.5 > gpurun_out/ab_g_nopf_$r.log 2>&1
GL_LIB=paper_2109_01611_b200/_ab/libgpulet_oldexec.so timeout 300 python tools/serve_ab.py --xs 2.27,2.5 > gpurun_out/ab_g_old_$r.log 2>&1
done
for m in resnet50:32 resnet50:15 lenet5:24; do mm=${m%:*}; b=${m#*:}
timeout 120 python tools/oneshot.py --model $mm --batch $b --json gpurun_out/trace_r1g_new_${mm}_b$b.json > /dev/null 2>&1
GL_LIB=paper_2109_01611_b200/_ab/libgpulet_nopf.so timeout 120 python tools/oneshot.py --model $mm --batch $b --json gpurun_out/trace_r1g_nopf_${mm}_b$b.json > /dev/null 2>&1
GL_LIB=paper_2109_01611_b200/_ab/libgpulet_oldexec.so timeout 120 python tools/oneshot.py --model $mm --batch $b --json gpurun_out/trace_r1g_old_${mm}_b$b.json > /dev/null 2>&1
done
echo done
