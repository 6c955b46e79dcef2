"""Per-point roofline of the latency profile (BASELINE metric
"per-gpu-let tensor/HBM % of roofline"): for every (model, batch, gpu-let size)
row of profiles/profile_b200.csv, the achieved tensor throughput (the method's
FLOPs of that batch, gl_model_cost, / the measured latency) against the
gpu-let's SM share of the sustained bf16 peak (n/148 x MEASURED_PEAKS
bf16_tflops_sustained), and the achieved algorithmic HBM rate (weights once +
the batch's inputs and outputs) against BW(n), the confined
copy bandwidth of that gpu-let size (K12 probe, gl_bw_probe).  The profile's
latencies are host-observed (R18), so short batches include the ~9-10 µs
service floor.  ResNet-50 rows are cfg2 (b 1-32 x {20,40,50,60,80,100} %).

    python tools/profile_roofline.py [--json profiles/profile_roofline_b200.json]
"""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthgen  # noqa: E402
from tools import common  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default="")
    ap.add_argument("--bytes", type=int, default=1 << 30)
    a = ap.parse_args()
    from paper_2109_01611_b200 import gpulet
    with open(os.path.join(common.ROOT, "MEASURED_PEAKS.json")) as f:
        peaks = json.load(f)
    p_sus = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    ctx = gpulet.Context(1)
    bw = {}
    for p in common.GRID:
        gbs, n = ctx.bw_probe(0, p, a.bytes, 5)
        bw[p] = (gbs, n)
    mids = {m: ctx.load_model(0, m, synthgen.weight_file(m)) for m in common.MODELS}
    cost = {}
    for m in common.MODELS:
        inb, outb = ctx.model_io(mids[m], 32)
        for b in range(1, 33):
            fl, wb = ctx.model_cost(mids[m], b)
            cost[m, b] = (fl, wb + b * (inb + outb) / 32)
    rows = []
    with open(common.PROFILE_CSV) as f:
        for r in csv.DictReader(f):
            m, b, p, n = r["model"], int(r["batch"]), int(r["partition_pct"]), int(r["sm_count"])
            lat = float(r["latency_us"])
            fl, by = cost[m, b]
            tf = fl / lat / 1e6
            gbs = by / lat / 1e3
            rows.append({"model": m, "batch": b, "pct": p, "sm": n, "latency_us": lat,
                         "tflops": round(tf, 2), "tensor_frac": round(tf / (p_sus * n / 148), 4),
                         "gbs": round(gbs, 1), "hbm_frac": round(gbs / bw[p][0], 4)})
    summ = {}
    for m in common.MODELS:
        rr = [r for r in rows if r["model"] == m]
        best = max(rr, key=lambda r: r["tensor_frac"])
        summ[m] = {"best_tensor_frac": best["tensor_frac"], "at": [best["batch"], best["pct"]],
                   "b32_100pct_tensor_frac": next(r["tensor_frac"] for r in rr if r["batch"] == 32 and r["pct"] == 100),
                   "b1_100pct_hbm_frac": next(r["hbm_frac"] for r in rr if r["batch"] == 1 and r["pct"] == 100)}
        print(m, json.dumps(summ[m]), flush=True)
    out = {"peak_tflops_sustained": p_sus, "bw_probe_gbs": {str(p): round(v[0], 1) for p, v in bw.items()},
           "sm": {str(p): v[1] for p, v in bw.items()}, "summary": summ, "rows": rows,
           "note": "latencies are host-observed (R18); FLOPs are the method's (real K); bytes = weights once + "
                   "the batch's inputs and outputs"}
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
