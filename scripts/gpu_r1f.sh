mkdir -p gpurun_out
timeout 300 python tools/serve_ab.py > gpurun_out/ab_new.log 2>&1
GL_LIB=paper_2109_01611_b200/_ab/libgpulet_oldexec.so timeout 300 python tools/serve_ab.py > gpurun_out/ab_old.log 2>&1
timeout 300 python tools/serve_ab.py > gpurun_out/ab_new2.log 2>&1
echo done
