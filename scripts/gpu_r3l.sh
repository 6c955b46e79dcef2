mkdir -p gpurun_out
for rep in 1 2; do
for g in "5 20" "10 20" "15 10" "2 1000"; do set -- $g
  GL_GUARD_MIN_US=$1 GL_GUARD_DIV=$2 timeout 300 python tools/serve_ab.py --xs 3.2,3.7,4.2,4.6 --secs 0.5 > gpurun_out/guard_r3l_${1}_${2}_$rep.log 2>&1
done; done
echo done
