mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do
for mb in resnet50:32 resnet50:8 vgg16:32 bert_base:32 googlenet:32; do m=${mb%:*}; b=${mb#*:}
  for bn in 0 128; do
    timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --bn $bn --json gpurun_out/bnab_${m}_b${b}_bn${bn}_r$rep.json > /dev/null 2>&1
  done
done
done
python - <<'PY'
import json, glob, statistics
rows = {}
for f in glob.glob("gpurun_out/bnab_*_r*.json"):
    k = f.split("bnab_")[1].rsplit("_r", 1)[0]
    rows.setdefault(k, []).append(json.load(open(f))["total_us"])
for k in sorted(rows):
    print(f"{k:32s} median {statistics.median(rows[k]):8.1f}  {sorted(rows[k])}")
PY
