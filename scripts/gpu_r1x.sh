mkdir -p gpurun_out
for rep in 1 2 3; do for v in 0 1 2; do for mb in resnet50:32 resnet50:15 vgg16:32 bert_base:32; do m=${mb%:*}; b=${mb#*:}
  if [ $v = 2 ]; then export GL_DATAFLOW_UNSAFE_REUSE=1; D=1; else unset GL_DATAFLOW_UNSAFE_REUSE; D=$v; fi
  GL_DATAFLOW=$D timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --json gpurun_out/ab_x_df${v}_${m}_b${b}_r$rep.json > /dev/null 2>&1
done; done; done
unset GL_DATAFLOW_UNSAFE_REUSE
python - <<PY > gpurun_out/ab_x.log
import json, glob, statistics
rows = {}
for f in glob.glob("gpurun_out/ab_x_*_r*.json"):
    k = f.split("ab_x_")[1].rsplit("_r", 1)[0]
    rows.setdefault(k, []).append(json.load(open(f))["total_us"])
for k in sorted(rows, key=lambda k: (k.split("_", 1)[1], k)):
    print(f"{k:34s} median {statistics.median(rows[k]):8.1f}  {sorted(rows[k])}")
PY
echo done
