mkdir -p gpurun_out
for rep in 1 2; do for sp in 0 1; do for mb in resnet50:8 resnet50:15 bert_base:8 googlenet:8 vgg16:8; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --split $sp --json gpurun_out/ab_f_s${sp}_${m}_b${b}_r$rep.json > /dev/null 2>&1
done; done; done
python - <<PY > gpurun_out/ab_f.log
import json, glob, statistics
rows = {}
for f in glob.glob("gpurun_out/ab_f_*_r*.json"):
    k = f.split("ab_f_")[1].rsplit("_r", 1)[0]
    d = json.load(open(f))
    rows.setdefault(k, []).append((d["total_us"], d["steps"]))
for k in sorted(rows, key=lambda k: (k.split("_", 1)[1], k)):
    print(f"{k:34s} median {statistics.median(r[0] for r in rows[k]):8.1f} steps {rows[k][0][1]}")
PY
echo done
