"""One-shot executor launches of one model batch (for ncu capture and the
per-step trace): `python tools/oneshot.py --model resnet50 --batch 32 --reps 3`.
Prints per-step device durations with each step's algorithmic FLOPs/bytes."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthgen  # noqa: E402
from tools import common  # noqa: E402

OPS = {1: "gemm", 2: "dwconv", 3: "maxpool", 4: "avgpool", 5: "lenet", 6: "embed_ln", 7: "layernorm",
       8: "attention", 9: "softmax", 10: "splitk_final"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--n_sm", type=int, default=0)
    ap.add_argument("--json", default="")
    ap.add_argument("--flags", type=int, default=0, help="executor dbg_flags (tuning experiments)")
    ap.add_argument("--split", type=int, default=0, help="force split-K count when building programs (tuning)")
    ap.add_argument("--bn", type=int, default=0, help="force the UMMA N tile when building programs (tuning)")
    ap.add_argument("--sm-target", type=int, default=0, help="SM count the tile decomposition targets (tuning)")
    a = ap.parse_args()
    import torch
    from paper_2109_01611_b200 import gpulet
    ctx = gpulet.Context(1)
    if a.flags:
        gpulet.Context.set_tuning(2, a.flags)
    if a.split:
        gpulet.Context.set_tuning(1, a.split)
    if a.bn:
        gpulet.Context.set_tuning(0, a.bn)
    if a.sm_target:
        gpulet.Context.set_tuning(5, a.sm_target)
    mid = ctx.load_model(0, a.model, synthgen.weight_file(a.model))
    x = common.device_input(a.model, a.batch)
    y = torch.empty(ctx.model_io(mid, a.batch)[1] // 4, device="cuda")
    runs = [ctx.run_once(mid, a.batch, x, y, a.n_sm, True, roles=True) for _ in range(a.reps)]
    roles = runs[-1][1]
    runs = [r[0] for r in runs]
    info = ctx.program_info(mid, a.batch)
    best = [min(r[i] for r in runs) for i in range(len(info))]
    tot = sum(best)
    rows = []
    for i, (t, n, f, b) in enumerate(info):
        rows.append({"step": i, "op": OPS.get(t, t), "ops": n, "us": round(best[i] / 1e3, 2), "gflop": round(f / 1e9, 3),
                     "mb": round(b / 1e6, 2), "tflops": round(f / max(best[i], 1) / 1e3, 1),
                     "gbs": round(b / max(best[i], 1), 1),
                     # CTA 0 role stamps (us from step start): prod start/end, mma first/last, epi first/end, bar in/out
                     "roles_us": [None if v is None else round(v / 1e3, 2) for v in roles[i]]})
    fl = sum(r[2] for r in info)
    summary = {"model": a.model, "batch": a.batch, "steps": len(info), "total_us": round(tot / 1e3, 1),
               "tflops": round(fl / tot / 1e3, 1), "rows": rows}
    print(json.dumps({k: v for k, v in summary.items() if k != "rows"}))
    for r in sorted(rows, key=lambda r: -r["us"])[:12]:
        print(r)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(summary, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
