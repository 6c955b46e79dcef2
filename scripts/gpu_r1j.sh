mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1j.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1j.log
bash scripts/ab_oneshot.sh j paper_2109_01611_b200/_ab/libgpulet_A.so paper_2109_01611_b200/libgpulet.so > gpurun_out/ab_j.log 2>&1
echo done
