D=paper_2109_01611_b200/_ab
mkdir -p gpurun_out
GL_LIB=$D/libgpulet_L.so timeout 300 python tools/_bert_err_tmp.py > gpurun_out/bert_err.log 2>&1
GL_LIB=$D/libgpulet_M.so timeout 300 python tools/_bert_err_tmp.py >> gpurun_out/bert_err.log 2>&1
