mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_models.py tests/test_gpu_serve.py -m gpu -q -x > gpurun_out/gputests_r1w.log 2>&1; echo "rc=$?" >> gpurun_out/gputests_r1w.log
for rep in 1 2 3; do for v in 0 1; do for mb in resnet50:32 resnet50:15 resnet50:1 bert_base:32 vgg16:32; do m=${mb%:*}; b=${mb#*:}
  GL_DATAFLOW=$v timeout 120 python tools/oneshot.py --model $m --batch $b --reps 5 --json gpurun_out/ab_w_df${v}_${m}_b${b}_r$rep.json > /dev/null 2>&1
done; done; done
python - <<PY > gpurun_out/ab_w.log
import json, glob, statistics
rows = {}
for f in glob.glob("gpurun_out/ab_w_*_r*.json"):
    k = f.split("ab_w_")[1].rsplit("_r", 1)[0]
    rows.setdefault(k, []).append(json.load(open(f))["total_us"])
for k in sorted(rows, key=lambda k: (k.split("_", 1)[1], k)):
    print(f"{k:34s} median {statistics.median(rows[k]):8.1f}  {sorted(rows[k])}")
PY
echo done
