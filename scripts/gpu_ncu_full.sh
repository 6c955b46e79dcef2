# One ncu --set full capture of a one-shot executor launch (tools/oneshot.py), with
# source correlation, plus local-memory counters.   bash scripts/gpu_ncu_full.sh TAG model batch
TAG=$1; M=${2:-resnet50}; B=${3:-32}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gl_executor -c 1 -f -o gpurun_out/ncu_${TAG}_${M}_b${B} python tools/oneshot.py --model $M --batch $B --reps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --metrics l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum,smsp__inst_executed_op_local_ld.sum,smsp__inst_executed_op_local_st.sum,gpu__time_duration.sum --clock-control none -k regex:gl_executor -c 1 --csv --log-file gpurun_out/ncu_local_${TAG}.csv python tools/oneshot.py --model $M --batch $B --reps 1 > gpurun_out/ncu_local_$TAG.log 2>&1
