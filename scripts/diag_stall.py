"""Diagnostic: where do the ms-scale LeNet-5 latency outliers of the game headline
come from?  Serves a LeNet-only lane (20 % gpu-let) at ~10 k req/s through
gl_serve for a few seconds while a Python thread spins on perf_counter and
records every host gap > 200 µs (a stall of the whole process: descheduling,
cgroup throttling, fork of a sampler).  Variants: plain; with an nvidia-smi
subprocess sampler every 200 ms (bench's old clock sampler); with an in-process
NVML sampler; with the frontend SCHED_FIFO (gl_set_tuning(7, 1)).  Prints, per
variant, the latency outliers (> 1 ms) and the host gaps."""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def spin(stop, gaps):
    last = time.perf_counter()
    while not stop.is_set():
        now = time.perf_counter()
        if now - last > 200e-6:
            gaps.append((last, (now - last) * 1e6))
        last = now


def smi_sampler(stop):
    while not stop.is_set():
        subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader"], capture_output=True)
        stop.wait(0.2)


def nvml_sampler(stop):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        stop.wait(0.2)


def main():
    import bench
    from paper_2109_01611_b200 import gpulet
    from tools import common
    ctx = gpulet.Context(1)
    srv = bench.Server(ctx, 0, False)
    rates, dump, ok = srv.plan("game", "gpulet", 1, 1.5)
    my = srv.setup(dump, 0)
    my = [r if i == 0 else 0 for i, r in enumerate(my)]   # LeNet only
    out = {}
    for variant in ("plain", "smi", "nvml", "fifo", "plain2"):
        if variant == "fifo":
            gpulet.Context.set_tuning(7, 1)
        stop, gaps = threading.Event(), []
        th = [threading.Thread(target=spin, args=(stop, gaps), daemon=True)]
        if variant == "smi":
            th.append(threading.Thread(target=smi_sampler, args=(stop,), daemon=True))
        if variant == "nvml":
            th.append(threading.Thread(target=nvml_sampler, args=(stop,), daemon=True))
        for t in th:
            t.start()
        res = []
        for r in range(4):
            t, m = bench.poisson_trace(my, 0.5, 9000 + r)
            t0 = time.perf_counter()
            lat = ctx.serve(srv.lanes, len(common.MODELS), t, m, srv.slo)
            big = [(round(float(t[i]) / 1e3, 2), int(lat[i])) for i in np.nonzero((lat > 1000) | (lat < 0))[0]]
            res.append({"n": int(len(lat)), "viol": int(((lat < 0) | (lat > srv.slo[0])).sum()),
                        "p999": float(np.percentile(lat[lat >= 0], 99.9)), "outliers_ms_lat": big[:10],
                        "n_outliers": len(big), "t0": t0})
        stop.set()
        for t in th:
            t.join(timeout=2)
        if variant == "fifo":
            gpulet.Context.set_tuning(7, 0)
        g = [(round(a, 4), round(d)) for a, d in gaps]
        out[variant] = {"runs": res, "host_gaps_over_200us": len(g), "max_gap_us": max([d for _a, d in g] or [0]),
                        "gaps_over_1ms": [d for _a, d in g if d > 1000][:20]}
        print(variant, json.dumps({k: v for k, v in out[variant].items() if k != "runs"}),
              [(x["viol"], x["n"], x["n_outliers"], round(x["p999"])) for x in res], flush=True)
    srv.teardown()
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
