"""Serving A/B check (tuning tool): violation fraction of the game/gpulet plan at
fixed rate multipliers, plus one-shot LeNet/ResNet latencies, for the library
named by GL_LIB (default: the in-tree build).
    GL_LIB=... python tools/serve_ab.py --xs 1.9,2.27 --secs 0.5"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--xs", default="1.9,2.27")
    ap.add_argument("--secs", type=float, default=0.5)
    ap.add_argument("--scenario", default="game")
    ap.add_argument("--mode", default="gpulet")
    a = ap.parse_args()
    import bench
    import torch
    from paper_2109_01611_b200 import gpulet
    from tools import common
    ctx = gpulet.Context(1)
    srv = bench.Server(ctx, 0, False)
    out = {"lib": os.environ.get("GL_LIB", "in-tree")}
    for m, b in (("lenet5", 24), ("resnet50", 15)):
        d = [sum(ctx.run_once(srv.mids[m], b, srv.x[m, 0], srv.y[m, 0], 0, True)) / 1e3 for _ in range(5)]
        out[f"{m}_b{b}_us"] = round(sorted(d)[2], 1)
    for x in [float(v) for v in a.xs.split(",")]:
        rates, dump, ok = srv.plan(a.scenario, a.mode, 1, x)
        my = srv.setup(dump, 0)
        ws = [srv.window(my, a.secs, 77 + i) for i in range(2)]
        srv.teardown()
        out[f"x{x}"] = {"viol": round(sum(w["viol"] for w in ws) / max(1, sum(w["arrivals"] for w in ws)), 4),
                        "per": {k: (v["viol"], v["p99_us"]) for k, v in ws[-1]["per"].items()}}
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
