mkdir -p gpurun_out
GL_DATAFLOW_LOG=1 timeout 120 python tools/oneshot.py --model resnet50 --batch 8 > gpurun_out/df_log_r1v.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputests_r1v.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1v.log
L=paper_2109_01611_b200/libgpulet.so
cp $L /tmp/lib_df.so
for rep in 1 2 3; do for v in 0 1; do for mb in resnet50:32 resnet50:15 resnet50:8 resnet50:1 bert_base:32 vgg16:32 googlenet:8 ssd_mobilenet_v1:8; do m=${mb%:*}; b=${mb#*:}
  GL_DATAFLOW=$v timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --json gpurun_out/ab_v_df${v}_${m}_b${b}_r$rep.json > /dev/null 2>&1
done; done; done
python - <<PY > gpurun_out/ab_v.log
import json, glob, statistics
rows = {}
for f in glob.glob("gpurun_out/ab_v_*_r*.json"):
    k = f.split("ab_v_")[1].rsplit("_r", 1)[0]
    rows.setdefault(k, []).append(json.load(open(f))["total_us"])
for k in sorted(rows, key=lambda k: (k.split("_", 1)[1], k)):
    print(f"{k:34s} median {statistics.median(rows[k]):8.1f}  {sorted(rows[k])}")
PY
echo done
