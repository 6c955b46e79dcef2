mkdir -p gpurun_out
for pq in "50 50" "60 40" "80 20" "40 60" "20 80" "20 20" "40 40"; do timeout 60 python scripts/diag_pairs.py $pq >> gpurun_out/diag12.log 2>&1; done
echo "--- SLOT1_REM" >> gpurun_out/diag12.log
for pq in "50 50" "40 40"; do GL_SLOT1_REM=1 timeout 60 python scripts/diag_pairs.py $pq >> gpurun_out/diag12.log 2>&1; done
echo "--- FORWARD=9" >> gpurun_out/diag12.log
for pq in "50 50"; do GL_SLOT1_FORWARD=9 timeout 60 python scripts/diag_pairs.py $pq >> gpurun_out/diag12.log 2>&1; done
