"""Per-gpu-let roofline during co-runs (BASELINE metric
"per-gpu-let tensor/HBM % of roofline"), from the committed measurements: for
each co-run sample of profiles/corun_b200.csv (victim model, batch, gpu-let
size, partner, measured slowdown factor = co-run / solo device latency) the
victim's achieved tensor rate is its solo rate at that (model, batch, size)
(profiles/profile_roofline_b200.json: the method's FLOPs / the profiled
latency) divided by the factor, against the gpu-let's SM share of the
sustained bf16 peak; the HBM rate likewise against BW(n) of that size.
Per-gpu-let ncu counters cannot be taken during a co-run: ncu serialises
kernels and replays each one, and a gpu-let's executor is a persistent kernel.

    python tools/corun_roofline.py [--json profiles/corun_roofline_b200.json]
"""
import argparse
import csv
import json
import os
import statistics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default=os.path.join(ROOT, "profiles", "corun_roofline_b200.json"))
    a = ap.parse_args()
    with open(os.path.join(ROOT, "profiles", "profile_roofline_b200.json")) as f:
        pr = json.load(f)
    solo = {(r["model"], r["batch"], r["pct"]): r for r in pr["rows"]}
    peak, bw = pr["peak_tflops_sustained"], {int(k): v for k, v in pr["bw_probe_gbs"].items()}
    rows = []
    with open(os.path.join(ROOT, "profiles", "corun_b200.csv")) as f:
        for r in csv.DictReader(f):
            m, b, p = r["victim"], int(r["vb"]), int(r["vp"])
            s = solo[(m, b, p)]
            fac = float(r["factor"])
            tf = s["tflops"] / fac
            gbs = s["gbs"] / fac
            rows.append({"victim": m, "batch": b, "pct": p, "sm": s["sm"], "partner": r["partner"], "partner_batch": int(r["pb"]),
                         "partner_pct": int(r["pp"]), "factor": round(fac, 4), "tflops": round(tf, 2),
                         "tensor_frac": round(tf / (peak * s["sm"] / 148), 4), "gbs": round(gbs, 1),
                         "hbm_frac": round(gbs / bw[p], 4)})
    cfg3 = [r for r in rows if r["pct"] == 50 and r["partner_pct"] == 50 and
            {r["victim"], r["partner"]} == {"resnet50", "vgg16"}]
    summ = {}
    for m in sorted({r["victim"] for r in rows}):
        rr = [r for r in rows if r["victim"] == m]
        summ[m] = {"samples": len(rr), "tensor_frac_median": round(statistics.median(r["tensor_frac"] for r in rr), 4),
                   "tensor_frac_max": max(r["tensor_frac"] for r in rr),
                   "factor_median": round(statistics.median(r["factor"] for r in rr), 4)}
    out = {"peak_tflops_sustained": peak, "bw_probe_gbs": pr["bw_probe_gbs"], "summary": summ,
           "cfg3_resnet50_vgg16_50_50": cfg3, "rows": rows,
           "note": "co-run rate = solo rate (method FLOPs / profiled host-observed latency) / measured co-run factor"}
    with open(a.json, "w") as f:
        json.dump(out, f, indent=1)
    for r in sorted(cfg3, key=lambda r: (r["victim"], r["batch"], r["partner_batch"])):
        if r["batch"] == r["partner_batch"]:
            print(f"cfg3 {r['victim']:9s} b{r['batch']:2d} next to {r['partner']} b{r['partner_batch']:2d}: "
                  f"factor {r['factor']:.3f}, {r['tflops']:7.1f} TFLOP/s = {100 * r['tensor_frac']:5.1f} % of its 74-SM share, "
                  f"{r['gbs']:7.1f} GB/s = {100 * r['hbm_frac']:4.1f} % of BW(74)")
    print(json.dumps(summ))


if __name__ == "__main__":
    main()
