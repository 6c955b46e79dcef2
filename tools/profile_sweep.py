"""Latency profiler sweep L(b, p) on a B200 (PAPER.md P:226-233,
P:370): every model x batch x gpu-let size, warm back-to-back batches on a
solo gpu-let, the 90th percentile of the host-observed service latency (submit ->
completion seen by gl_poll, R18) over --reps batches, written to
profiles/profile_b200.csv with solo utilisation features (a3).

Utilisation features (reading, DESIGN.md §2 R-stat): the paper reads L2 and
DRAM utilisation from Nsight Compute.  Here each (m, b, p) row
carries the program's algorithmic traffic over its measured latency, relative
to whole-GPU peaks: mem = weight+I/O bytes / (L x HBM peak), l2 = all operand
bytes / (L x L2 peak); ncu-measured values can replace them without changing
the scheduler.

    python tools/profile_sweep.py [--batches all|pow2] [--reps 50] [--warmup 3] [--quantile 0.9] [--keep-stats CSV]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import synthgen  # noqa: E402
from tools import common  # noqa: E402

HBM_GBS = 6451.8
L2_GBS = 20000.0   # effective L2 bandwidth used to normalise the l2 feature


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="all")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=common.PROFILE_CSV)
    ap.add_argument("--models", default=",".join(common.MODELS))
    ap.add_argument("--quantile", type=float, default=0.9,
                    help="L(b, p) = this quantile of the reps host-observed service latencies (R18: 0.9)")
    ap.add_argument("--keep-stats", default="",
                    help="keep the l2_util / mem_bw_util columns of this profile CSV (ncu-measured, a3)")
    a = ap.parse_args()
    import torch
    from paper_2109_01611_b200 import gpulet

    batches = list(range(1, 33)) if a.batches == "all" else list(common.STAT_B)
    models = a.models.split(",")
    ctx = gpulet.Context(1)
    mids = {m: ctx.load_model(0, m, synthgen.weight_file(m)) for m in common.MODELS}
    xs = {m: common.device_input(m, 32) for m in common.MODELS}
    ys = {m: torch.empty(ctx.model_io(mids[m], 32)[1] // 4, device="cuda") for m in common.MODELS}
    M = len(common.MODELS)
    lat = [[[0] * 6 for _ in range(32)] for _ in range(M)]
    l2 = [[[0.0] * 6 for _ in common.STAT_B] for _ in range(M)]
    mem = [[[0.0] * 6 for _ in common.STAT_B] for _ in range(M)]
    nsm = [0] * 6
    t0 = time.time()
    for gi, p in enumerate(common.GRID):
        (gid, n), = ctx.create_gpulets(0, [p])
        nsm[gi] = n
        for mi, m in enumerate(common.MODELS):
            if m not in models:
                continue
            for b in batches:
                us = ctx.profile_tail(gid, mids[m], b, xs[m], ys[m], a.warmup, a.reps, a.quantile)[1]
                lat[mi][b - 1][gi] = int(np.ceil(us))
            print(f"p={p} ({n} SMs) {m}: " + " ".join(str(lat[mi][b - 1][gi]) for b in batches), flush=True)
        ctx.destroy_gpulet(gid)
    # fill unmeasured batches with the next measured one (S:67 ceiling rule)
    for mi in range(M):
        for gi in range(6):
            nxt = None
            for b in range(32, 0, -1):
                if b in batches:
                    nxt = lat[mi][b - 1][gi]
                elif nxt is not None:
                    lat[mi][b - 1][gi] = nxt
    for mi, m in enumerate(common.MODELS):
        for si, b in enumerate(common.STAT_B):
            info = ctx.program_info(mids[m], b)
            tot_bytes = sum(s[3] for s in info)
            fl, wb = ctx.model_cost(mids[m], b)
            inb, outb = ctx.model_io(mids[m], b)
            for gi in range(6):
                L = max(lat[mi][b - 1][gi], 1) * 1e-6
                mem[mi][si][gi] = min(1.0, (wb + inb + outb) / (L * HBM_GBS * 1e9))
                l2[mi][si][gi] = min(1.0, tot_bytes / (L * L2_GBS * 1e9))
    if a.keep_stats:
        kept = common.load_profile(a.keep_stats)
        l2, mem = kept["l2"], kept["mem"]
    common.write_profile_csv(a.out, lat, nsm, l2, mem)
    print(json.dumps({"profile": a.out, "quantile": a.quantile, "reps": a.reps, "seconds": round(time.time() - t0, 1), "sm_count": nsm}))
    ctx.close()


if __name__ == "__main__":
    main()
