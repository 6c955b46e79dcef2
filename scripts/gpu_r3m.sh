mkdir -p gpurun_out
for rep in 1 2; do
for g in "5 20" "0 1000000" "1 1000" "2 1000" "3 1000"; do set -- $g
  GL_GUARD_MIN_US=$1 GL_GUARD_DIV=$2 timeout 300 python tools/serve_ab.py --xs 2.5,3.2,3.7,4.2 --secs 0.5 > gpurun_out/guard_r3m_${1}_${2}_$rep.log 2>&1
done; done
echo done
