# A/B/... one-shot traces on one box, interleaved, 3 reps:
#   VARIANTS="A=path/libA.so B=path/libB.so" bash scripts/ab_oneshot.sh TAG [model:batch ...]
TAG=$1; shift 1
MODELS=${@:-resnet50:32 resnet50:8 resnet50:15 bert_base:32}
mkdir -p gpurun_out
for rep in 1 2 3; do
  for vl in $VARIANTS; do v=${vl%%=*}; L=${vl#*=}
    for mb in $MODELS; do m=${mb%:*}; b=${mb#*:}
      GL_LIB=$L timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --json gpurun_out/ab_${TAG}_${v}_${m}_b${b}_r$rep.json > /dev/null 2>&1
    done
  done
done
python - <<PY
import json, glob, statistics
rows = {}
for f in glob.glob("gpurun_out/ab_${TAG}_*_r*.json"):
    k = f.split("ab_${TAG}_")[1].rsplit("_r", 1)[0]
    rows.setdefault(k, []).append(json.load(open(f))["total_us"])
for k in sorted(rows, key=lambda k: (k.split("_", 1)[1], k)):
    print(f"{k:32s} median {statistics.median(rows[k]):8.1f}  {sorted(rows[k])}")
PY
