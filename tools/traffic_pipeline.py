"""`traffic` as a two-stage pipeline on one B200 (PAPER.md
P:788-790: SSD-MobileNet detects objects, GoogLeNet and VGG-16 recognise them).

Per repetition, on device-resident synthetic inputs:
  stage 1  SSD-MobileNet-V1 batch B through the executor (gl_run_once, whole GPU)
  hand-off gl_ssd_detect (decode + per-class NMS + merge, R27) and
           gl_crop_resize (the first K detections per image -> 224 x 224 crops)
  stage 2  GoogLeNet and VGG-16 on the B*K crops (gl_run_once each)
Device times: executor %globaltimer for the model stages, CUDA events on the
launching stream for the hand-off kernels; median over --reps.  With random
weights the detector's scores are near-uniform, so --score-thr is a workload
knob (the number of detections is reported), not an accuracy claim.

    python tools/traffic_pipeline.py [--batch 8] [--per-img 4] [--reps 20] [--json out.json]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthgen  # noqa: E402
from tools import common  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--per-img", type=int, default=4)
    ap.add_argument("--score-thr", type=float, default=0.06)
    ap.add_argument("--iou-thr", type=float, default=0.45)
    ap.add_argument("--top-k", type=int, default=200)
    ap.add_argument("--max-det", type=int, default=100)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    import torch
    from paper_2109_01611_b200 import gpulet
    B, K = a.batch, a.per_img
    assert B * K <= 32, "recogniser batch must be <= 32 (P:766)"
    ctx = gpulet.Context(1)
    mids = {m: ctx.load_model(0, m, synthgen.weight_file(m)) for m in ("ssd_mobilenet_v1", "googlenet", "vgg16")}
    x = common.device_input("ssd_mobilenet_v1", B)
    heads = torch.empty(ctx.model_io(mids["ssd_mobilenet_v1"], B)[1] // 4, device="cuda")
    loc, conf = heads[:B * 3000 * 4], heads[B * 3000 * 4:]
    det = torch.empty((B, a.max_det, 7), device="cuda")
    cnt = torch.empty(B, dtype=torch.int32, device="cuda")
    ws = torch.empty(gpulet.ssd_detect_workspace(B, a.top_k), dtype=torch.uint8, device="cuda")
    crops = torch.empty((B * K, 224, 224, 8), dtype=torch.bfloat16, device="cuda")
    ys = {m: torch.empty(ctx.model_io(mids[m], B * K)[1] // 4, device="cuda") for m in ("googlenet", "vgg16")}
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    rows = []
    for rep in range(a.reps + 2):
        t_ssd = sum(ctx.run_once(mids["ssd_mobilenet_v1"], B, x, heads, 0, True)) / 1e3
        ev[0].record(stream)
        gpulet.ssd_detect(loc, conf, B, det, cnt, ws, a.score_thr, a.iou_thr, a.top_k, a.max_det, stream.cuda_stream)
        ev[1].record(stream)
        gpulet.crop_resize(x, B, 300, 300, det, cnt, a.max_det, K, crops, 224, 224, 8, stream.cuda_stream)
        ev[2].record(stream)
        torch.cuda.synchronize()
        t_det, t_crop = ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3
        t_g = sum(ctx.run_once(mids["googlenet"], B * K, crops, ys["googlenet"], 0, True)) / 1e3
        t_v = sum(ctx.run_once(mids["vgg16"], B * K, crops, ys["vgg16"], 0, True)) / 1e3
        if rep >= 2:
            rows.append((t_ssd, t_det, t_crop, t_g, t_v))
    med = [statistics.median(r[i] for r in rows) for i in range(5)]
    counts = cnt.cpu().tolist()
    out = {"batch": B, "per_img": K, "recogniser_batch": B * K, "score_thr": a.score_thr, "iou_thr": a.iou_thr,
           "top_k": a.top_k, "max_det": a.max_det, "detections_per_image": counts,
           "median_us": {"ssd": round(med[0], 1), "ssd_detect": round(med[1], 1), "crop_resize": round(med[2], 1),
                         "googlenet": round(med[3], 1), "vgg16": round(med[4], 1)},
           "handoff_frac_of_pipeline": round((med[1] + med[2]) / sum(med), 4),
           "pipeline_us_sequential": round(sum(med), 1),
           "note": "model stages on 148 SMs one after another; on gpu-lets the two recognisers run side by side"}
    print(json.dumps(out))
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
