mkdir -p gpurun_out
for rep in 1 2; do for nsm in 96 56; do for t in 0 $nsm; do for mb in resnet50:15 resnet50:32 googlenet:15 ssd_mobilenet_v1:8 vgg16:8; do m=${mb%:*}; b=${mb#*:}
  timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --n_sm $nsm --sm-target $t --json gpurun_out/smt_${nsm}_t${t}_${m}_b${b}_r$rep.json > /dev/null 2>&1
done; done; done; done
python - <<PY > gpurun_out/smt.log
import json, glob, statistics
rows = {}
for f in glob.glob("gpurun_out/smt_*_r*.json"):
    k = f.split("smt_")[1].rsplit("_r", 1)[0]
    rows.setdefault(k, []).append(json.load(open(f))["total_us"])
for k in sorted(rows):
    print(f"{k:40s} median {statistics.median(rows[k]):8.1f}")
PY
echo done
