"""Measurement gaps of SURVEY §8(d) (one B200):

* K12: the HBM roof BW(n) of every gpu-let size, a 16-B stream copy confined to
  the size's green context (gl_bw_probe; D0 "BW(n) is measured, not assumed");
* cfg1: the executor floor (an empty program through the ring, gl_floor) on
  every size, and LeNet-5 b = 32 on a 100 % gpu-let: device latency median / p99
  of 1,000 back-to-back batches after 10 warm-up, and the host submit -> poll
  round trip (gl_profile).

    python tools/measure_extras.py --json profiles/extras_b200.json
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import synthgen  # noqa: E402
from tools import common  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", default="")
    ap.add_argument("--bytes", type=int, default=1 << 30)
    a = ap.parse_args()
    import torch
    from paper_2109_01611_b200 import gpulet
    ctx = gpulet.Context(1)
    mid = ctx.load_model(0, "lenet5", synthgen.weight_file("lenet5"))
    out = {"bw_probe": {}, "floor": {}, "cfg1_lenet5_b32": {}}
    for p in common.GRID:
        gbs, n = ctx.bw_probe(0, p, a.bytes, 10)
        out["bw_probe"][str(p)] = {"sm": n, "gbs": round(gbs, 1)}
        print(f"BW({n} SMs, {p}%) = {gbs:.1f} GB/s", flush=True)
    med, p99 = ctx.publish_probe(0, 1000)
    out["publish_probe"] = {"h2d_64B_copy_us_median": round(med, 2), "p99": round(p99, 2),
                            "note": "host round trip of publishing one work descriptor into device memory; "
                                    "compare with the floor's whole host round trip through the mapped ring"}
    print(f"publish 64 B descriptor by H2D copy: median {med:.2f} us, p99 {p99:.2f} us", flush=True)
    for p in common.GRID:
        (gid, n), = ctx.create_gpulets(0, [p])
        h, d = ctx.floor(gid, 20, 500)
        out["floor"][str(p)] = {"sm": n, "host_round_trip_us": round(h, 2), "device_us": round(d, 2)}
        print(f"floor {p}% ({n} SMs): host {h:.2f} us, device {d:.2f} us", flush=True)
        ctx.destroy_gpulet(gid)
    # device buffers before the executor: a whole-GPU executor leaves no SM for torch's kernels
    x = common.device_input("lenet5", 32)
    y = torch.empty(ctx.model_io(mid, 32)[1] // 4, device="cuda")
    torch.cuda.synchronize()
    (gid, n), = ctx.create_gpulets(0, [100])
    print("cfg1: gpu-let created", flush=True)
    tickets = [ctx.submit_batch(gid, mid, x, y, 32, 5.0) for _ in range(10)]
    for t in tickets:
        ctx.wait(t)
    print("cfg1: warm-up done", flush=True)
    dev = []
    for _ in range(1000):
        c = ctx.wait(ctx.submit_batch(gid, mid, x, y, 32, 5.0))
        dev.append((c.t_end_ns - c.t_start_ns) / 1e3)
    print("cfg1: 1000 batches done", flush=True)
    host = ctx.profile(gid, mid, 32, x, y, 10, 200)
    dev = np.asarray(dev)
    out["cfg1_lenet5_b32"] = {"sm": n, "device_us_median": round(float(np.median(dev)), 2),
                              "device_us_p99": round(float(np.percentile(dev, 99)), 2),
                              "host_round_trip_us_median": round(host, 2), "batches": len(dev),
                              "fma_bound_us": "26.66 MFLOP / (148 SMs x 128 lanes x 2 FLOP x 1.965 GHz) = 0.36 us"}
    print(json.dumps(out["cfg1_lenet5_b32"]), flush=True)
    ctx.destroy_gpulet(gid)
    ctx.close()
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
