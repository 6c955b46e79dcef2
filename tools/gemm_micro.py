"""Per-op GEMM microbenchmark (tuning tool, GPU only).

Runs single-op conv / linear programs through the executor (gl_test_conv /
gl_test_gemm, warm + measured launch on the whole GPU), and prints device time,
TFLOP/s and the per-CTA tile timeline summary of the GEMM step:
  python tools/gemm_micro.py [--json out.json] [--bn 0,64,128] [--only name]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# name: (kind, args) ; conv args = N,H,W,C,Cout,KH,stride,pad ; gemm args = M,N,K
SHAPES = {
    "res_conv1": ("conv", (32, 224, 224, 8, 64, 7, 2, 3)),
    "res_l1_1x1_64": ("conv", (32, 56, 56, 64, 64, 1, 1, 0)),
    "res_l1_1x1_256to64": ("conv", (32, 56, 56, 256, 64, 1, 1, 0)),
    "res_l1_3x3_64": ("conv", (32, 56, 56, 64, 64, 3, 1, 1)),
    "res_l1_1x1_256": ("conv", (32, 56, 56, 64, 256, 1, 1, 0)),
    "res_l2_3x3_128": ("conv", (32, 28, 28, 128, 128, 3, 1, 1)),
    "res_l3_3x3_256": ("conv", (32, 14, 14, 256, 256, 3, 1, 1)),
    "res_l3_1x1_1024to256": ("conv", (32, 14, 14, 1024, 256, 1, 1, 0)),
    "res_l3_1x1_256to1024": ("conv", (32, 14, 14, 256, 1024, 1, 1, 0)),
    "res_l4_3x3_512": ("conv", (32, 7, 7, 512, 512, 3, 1, 1)),
    "vgg_3x3_64_224": ("conv", (32, 224, 224, 64, 64, 3, 1, 1)),
    "vgg_3x3_256_56": ("conv", (32, 56, 56, 256, 256, 3, 1, 1)),
    "vgg_3x3_512_28": ("conv", (32, 28, 28, 512, 512, 3, 1, 1)),
    "bert_ffn1": ("gemm", (4096, 3072, 768)),
    "bert_ffn2": ("gemm", (4096, 768, 3072)),
    "bert_qkv": ("gemm", (4096, 2304, 768)),
}


def bits(a):
    return np.ascontiguousarray(a.astype(np.float32)).view(np.uint32).__rshift__(16).astype(np.uint16)


def run(ctx, name, kind, args, rng):
    import torch
    from paper_2109_01611_b200 import gpulet
    if kind == "conv":
        N, H, W, C, Co, KH, s, p = args
        Ho, Wo = (H + 2 * p - KH) // s + 1, (W + 2 * p - KH) // s + 1
        x = torch.randn(N, H, W, C, device="cuda").clamp(-3, 3).to(torch.bfloat16)
        w = bits(rng.standard_normal((Co, KH, KH, C)) * np.sqrt(2.0 / (KH * KH * C)))
        b = bits(rng.uniform(-0.05, 0.05, Co))
        y = torch.empty(N, Ho, Wo, Co, device="cuda", dtype=torch.bfloat16)
        ctx.test_conv(0, x, w, b, y, N, H, W, C, Co, KH, s, p, 1, 1)
        flops = 2.0 * N * Ho * Wo * Co * KH * KH * C
        M, Nn, K = N * Ho * Wo, Co, KH * KH * C
    else:
        M, Nn, K = args
        x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = bits(rng.standard_normal((Nn, K)) * np.sqrt(2.0 / K))
        b = bits(rng.uniform(-0.05, 0.05, Nn))
        y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
        ctx.test_gemm(0, x, w, b, y, M, Nn, K, 1, 0, 1, 0, 1)
        flops = 2.0 * M * Nn * K
    ns, tl = gpulet.Context.test_stats()
    used = tl[:, :, 0] > 0
    ntiles = used.sum(1)
    epi = (tl[:, :, 3] - tl[:, :, 2]).astype(np.float64)[used] / 1e3
    mma = (tl[:, :, 1] - tl[:, :, 0]).astype(np.float64)[used] / 1e3
    first = tl[:, 0, 0][ntiles > 0].astype(np.float64) / 1e3
    first = first[first < 1e9]
    last = np.array([tl[c, n - 1, 3] for c, n in enumerate(ntiles) if n > 0], dtype=np.float64) / 1e3
    r = {"name": name, "M": M, "N": Nn, "K": K, "us": round(ns / 1e3, 2), "tflops": round(flops / ns / 1e3, 1),
         "tiles_per_cta": [int(ntiles.min()), int(ntiles.max())],
         "first_mma_us": [round(first.min(), 2), round(float(np.median(first)), 2), round(first.max(), 2)],
         "last_epi_end_us": [round(last.min(), 2), round(float(np.median(last)), 2), round(last.max(), 2)],
         "mma_us_p50_p90_max": [round(float(np.percentile(mma, q)), 2) for q in (50, 90, 100)],
         "epi_us_p50_p90_max": [round(float(np.percentile(epi, q)), 2) for q in (50, 90, 100)]}
    cta0 = [[round(v / 1e3, 2) for v in tl[0, i]] for i in range(int(ntiles[0]))]
    r["cta0"] = cta0[:12]
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default="")
    ap.add_argument("--bn", default="0")
    ap.add_argument("--split", default="0")
    ap.add_argument("--only", default="")
    ap.add_argument("--flags", default="0", help="executor dbg_flags sweep (tuning experiments)")
    a = ap.parse_args()
    from paper_2109_01611_b200 import gpulet
    ctx = gpulet.Context(1)
    gpulet.Context.set_tuning(3, 1)   # one warm-up launch before the measured one
    rng = np.random.default_rng(0)
    out = []
    for name, (kind, args) in SHAPES.items():
        if a.only and not any(o in name for o in a.only.split(",")):
            continue
        for bn in [int(v) for v in a.bn.split(",")]:
            for sp in [int(v) for v in a.split.split(",")]:
                for fl in [int(v) for v in a.flags.split(",")]:
                    gpulet.Context.set_tuning(0, bn)
                    gpulet.Context.set_tuning(1, sp)
                    gpulet.Context.set_tuning(2, fl)
                    try:
                        r = run(ctx, name, kind, args, rng)
                    except Exception as e:  # keep sweeping
                        r = {"name": name, "error": str(e)}
                    r["bn"], r["split"], r["flags"] = bn, sp, fl
                    print(json.dumps(r), flush=True)
                    out.append(r)
    for k in range(4):
        gpulet.Context.set_tuning(k, 0)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
