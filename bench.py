#!/usr/bin/env python
"""bench.py — SLO-satisfying req/s of mixed-model serving on gpu-lets (B200).

Workload (BASELINE.json configs[3], the metric's 1-GPU configuration).  The
config text names the paper's `game` scenario but lists six models; SURVEY D2
keeps both readings, so one run measures both:
  * headline `game`: app request = 6 LeNet-5 + 1 ResNet-50 (the paper's
    definition of game), on gpu-lets planned by the native scheduler;
  * `mix6`: the six models (LeNet-5, GoogLeNet, ResNet-50, SSD-MobileNet-V1,
    VGG-16, BERT-base) at equal rates (Table tab:particular-scenarios P:800-806
    extended with BERT), reported under "mix6";
  * the whole-GPU temporal-sharing baseline (SBP) built from the same
    kernels, on the same scenario, reported under "baseline_sbp".
SLOs follow the paper's rule SLO = 2 x solo latency at batch 32
applied to the measured B200 profile (profiles/profile_b200.csv); rates are the
paper's rates scaled to B200 (C4.3) times the largest multiplier for which the
scheduler (Alg. 1, gpulet+int by default) returns Schedulable.  The plan's
gpu-lets are created (green contexts + persistent executors) and every step
replays one duty-cycle round: each lane submits one batch of its planned batch
size, gpu-lets run concurrently, lanes on a gpu-let run FIFO.  A request counts
as SLO-satisfying when D (its lane's batch-building window) + (its batch's
completion - round start, device %globaltimer) <= its model's SLO.

  value    = SLO-satisfying requests of the K timed rounds / device time of the
             K rounds (first dequeue -> last completion), summed over ranks /
             max over ranks
  e2e      = the same through the public API with pinned host inputs copied
             H2D and outputs copied D2H inside every step (host wall clock)
  roofline = the dominant lane's program at its batch, one executor launch on
             the whole GPU, FLOPs / launch time vs the measured bf16 peak
Multi-GPU: one process per GPU (torchrun); each GPU serves its own copy of the
1-GPU plan (requests are independent: no collective on the data path), weak
scaling.  --impl reference times the CPU oracle (oracle/) on a bounded sample.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402

METRIC = "SLO-satisfying req/s (mixed-model serving on gpu-lets)"
UNIT = "req/s"
VERBOSE = False


def log(*a):
    if VERBOSE:
        print(*a, file=sys.stderr, flush=True)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu):
        self.gpu, self.rows, self.stop = gpu, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def init_dist(world, backend):
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group(backend=backend)
        return dist
    return None


# ----------------------------------------------------------------------------- oracle arm
def reference_arm(a, world, rank):
    """The CPU oracle (fp64 numpy forward) as it stands, one request per step,
    models cycled in canonical order (bounded sample of the same mixed workload)."""
    if rank != 0:
        return None
    from oracle import models as omodels
    ws = {m: synthgen.weights(m) for m in synthgen.MODELS}
    order = list(synthgen.MODELS)
    times = []
    for s in range(a.warmup + a.steps):
        m = order[s % len(order)]
        x = synthgen.model_input(m, 1, batch_id=s)
        t0 = time.perf_counter()
        omodels.forward(m, ws[m], x)
        if s >= a.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = a.steps / tot
    cores = os.cpu_count()
    return {"impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": UNIT, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1000 * tot / a.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "oracle forward, 1 request per step cycling the six models"},
            "cpu_baseline": {"value": round(val, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "1 request per step, models cycled in canonical order"},
            "e2e": {"value": round(val, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def cpu_baseline_sample():
    """Oracle on the host cores: one request of each of the six models (batch 1)."""
    from oracle import models as omodels
    t = 0.0
    for m in synthgen.MODELS:
        w = synthgen.weights(m)
        x = synthgen.model_input(m, 1)
        t0 = time.perf_counter()
        omodels.forward(m, w, x)
        t += time.perf_counter() - t0
    return {"value": round(len(synthgen.MODELS) / t, 4), "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": "one batch-1 request of each of the six models (fp64 numpy forward)"}


# ----------------------------------------------------------------------------- our arm
def plan_for(lat_env, l2, mem, slo, coeffs, mode, scenario):
    """Largest rate multiplier (bisection, 0.5 %) the native scheduler accepts."""
    from paper_2109_01611_b200 import gpulet
    from tools import common
    lo, hi = 0.0, 1.0
    while True:
        _d, ok = gpulet.schedule(common.MODELS, lat_env, l2, mem, slo, common.scenario_rates(scenario, slo, hi), 1,
                                 mode, coeffs)
        if not ok or hi > 1e6:
            break
        lo, hi = hi, hi * 2
    for _ in range(40):
        mid = (lo + hi) / 2
        _d, ok = gpulet.schedule(common.MODELS, lat_env, l2, mem, slo, common.scenario_rates(scenario, slo, mid), 1,
                                 mode, coeffs)
        lo, hi = (mid, hi) if ok else (lo, mid)
        if hi - lo < 0.005 * max(lo, 1e-9):
            break
    rates = common.scenario_rates(scenario, slo, lo)
    dump, ok = gpulet.schedule(common.MODELS, lat_env, l2, mem, slo, rates, 1, mode, coeffs)
    return lo, rates, dump, ok


def run_scenario(ctx, gpu, mids, prof, scenario, mode, steps, warmup, e2e_leg, dist=None, clocks=False):
    import torch
    from tools import common
    lat_env, l2, mem, slo, coeffs = prof
    x, rates, dump, ok = plan_for(lat_env, l2, mem, slo, coeffs, mode, scenario)
    gls, _verdict = common.parse_plan(dump)
    log(f"[{scenario}/{mode}] x={x:.4f} rates={rates}\n{dump}")
    # every device buffer exists before any executor starts (a device allocation
    # can synchronise the device and would wait behind a persistent kernel)
    lanes, made = [], {}
    used = [g for g in sorted(gls, key=lambda d: d["slot"]) if g["lanes"]]
    for g in used:
        for ln in g["lanes"]:
            m = ln["model"]
            mi = common.MODELS.index(m)
            lanes.append(dict(gid=None, slot=g["slot"], model=m, mid=mids[m], batch=ln["batch"], D=g["D_us"],
                              x=common.device_input(m, ln["batch"]),
                              y=torch.empty(ctx.model_io(mids[m], ln["batch"])[1] // 4, device="cuda"), slo=slo[mi]))
    hx = [common.host_input(ln["model"], ln["batch"]) for ln in lanes] if e2e_leg else []
    hy = [torch.empty(ln["y"].numel(), dtype=torch.float32).pin_memory() for ln in lanes] if e2e_leg else []
    cs = torch.cuda.Stream()
    torch.cuda.current_stream().synchronize()
    if not lanes:
        return {"value": 0.0, "rate_multiplier": x, "rates": rates, "plan": dump, "lanes": []}
    for g, (gid, nsm) in zip(used, ctx.create_gpulets(gpu, [g["size"] for g in used])):
        made[gid] = (g["size"], nsm)
        for ln in lanes:
            if ln["slot"] == g["slot"]:
                ln["gid"] = gid

    def round_once(collect):
        tickets = {ctx.submit_batch(ln["gid"], ln["mid"], ln["x"], ln["y"], ln["batch"], ln["slo"] / 1000.0): i
                   for i, ln in enumerate(lanes)}
        recs = []
        while len(recs) < len(lanes):
            recs += ctx.poll()
        if collect is not None:
            collect.append([(tickets[r.ticket], r.t_dequeue_ns, r.t_start_ns, r.t_end_ns) for r in recs])

    try:
        for _ in range(warmup):
            round_once(None)
        rounds = []
        if dist:
            dist.barrier()
        torch.cuda.current_stream().synchronize()
        clk = ClockSampler(gpu) if clocks else None
        if clk:
            clk.__enter__()
        t0 = time.perf_counter()
        for _ in range(steps):
            round_once(rounds)
        wall = time.perf_counter() - t0
        if clk:
            clk.__exit__()
        t_first = min(min(r[1] for r in rd) for rd in rounds)
        t_last = max(max(r[3] for r in rd) for rd in rounds)
        dev_s = (t_last - t_first) * 1e-9
        sat = tot = 0
        busy = {gid: 0 for gid in made}
        flops_g = {gid: 0.0 for gid in made}
        lane_time = [0] * len(lanes)
        for rd in rounds:
            start = min(r[1] for r in rd)
            for i, _tdq, ts, te in rd:
                ln = lanes[i]
                tot += ln["batch"]
                if ln["D"] + (te - start) / 1000.0 <= ln["slo"]:
                    sat += ln["batch"]
                busy[ln["gid"]] += te - ts
                flops_g[ln["gid"]] += ctx.model_cost(ln["mid"], ln["batch"])[0]
                lane_time[i] += te - ts
        e2e = None
        if e2e_leg:
            h2d = sum(t.numel() * t.element_size() for t in hx)
            d2h = sum(t.numel() * 4 for t in hy)
            e_sat = e_tot = 0
            t0 = time.perf_counter()
            for _ in range(steps):
                ts = time.perf_counter()
                with torch.cuda.stream(cs):
                    for ln, h in zip(lanes, hx):
                        ln["x"].copy_(h.view(ln["x"].dtype).view(ln["x"].shape), non_blocking=True)
                cs.synchronize()
                tickets = {ctx.submit_batch(ln["gid"], ln["mid"], ln["x"], ln["y"], ln["batch"]): i
                           for i, ln in enumerate(lanes)}
                done = 0
                while done < len(lanes):
                    for r in ctx.poll():
                        i = tickets[r.ticket]
                        with torch.cuda.stream(cs):
                            hy[i].copy_(lanes[i]["y"], non_blocking=True)
                        done += 1
                cs.synchronize()
                el_us = (time.perf_counter() - ts) * 1e6
                for ln in lanes:
                    e_tot += ln["batch"]
                    e_sat += ln["batch"] if ln["D"] + el_us <= ln["slo"] else 0
            e_wall = time.perf_counter() - t0
            e2e = {"value": round(e_sat / e_wall, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(d2h), "all_req_per_s": round(e_tot / e_wall, 2)}
    finally:
        for gid in list(made):
            ctx.destroy_gpulet(gid)
    dom = max(range(len(lanes)), key=lambda i: lane_time[i])
    return {"value": sat / dev_s, "sat": sat, "tot": tot, "dev_s": dev_s, "wall": wall, "rate_multiplier": x,
            "rates": rates, "plan": dump, "e2e": e2e, "clocks": clk.summary() if clk else None,
            "gpulets": [{"size": made[g][0], "sm": made[g][1]} for g in made],
            "lanes": [{"model": ln["model"], "batch": ln["batch"], "D_us": ln["D"]} for ln in lanes],
            "gpulet_tensor_frac": {str(g): round(flops_g[g] / max(busy[g] * 1e-9, 1e-12) / 1e12 /
                                                 (_peaks()[1] * made[g][1] / 148), 4) for g in made},
            "dominant": lanes[dom]}


def our_arm(a, world, rank, local, dist):
    import torch
    from paper_2109_01611_b200 import gpulet
    from tools import common
    from tools.dist_agg import aggregate

    torch.cuda.set_device(local)
    hbm, peak_burst, _peak_sus, peak_src = _peaks()
    ctx = gpulet.Context(local + 1)
    gpu = local
    mids = {m: ctx.load_model(gpu, m, synthgen.weight_file(m)) for m in common.MODELS}
    if not os.path.exists(common.PROFILE_CSV):
        raise SystemExit(f"missing {common.PROFILE_CSV}: run tools/profile_sweep.py on the GPU first")
    lat, l2, mem = common.read_profile_csv(common.PROFILE_CSV)
    lat_env = [common.envelope(lat[m]) for m in range(len(common.MODELS))]
    slo = common.slos_from(lat_env)
    prof = (lat_env, l2, mem, slo, common.load_coeffs())
    head = run_scenario(ctx, gpu, mids, prof, a.scenario, a.mode, a.steps, a.warmup, not a.no_e2e, dist, clocks=True)
    extra = {}
    if not a.headline_only:
        for key, scen, mode in (("baseline_sbp", a.scenario, "sbp"), ("mix6", "mix6", a.mode),
                                ("mix6_baseline_sbp", "mix6", "sbp")):
            r = run_scenario(ctx, gpu, mids, prof, scen, mode, a.steps, a.warmup, False)
            extra[key] = {"value": round(r["value"], 2), "scenario": scen, "mode": mode,
                          "rate_multiplier": round(r["rate_multiplier"], 4), "rates_req_s": r["rates"],
                          "lanes": r["lanes"]}
    # roofline: the dominant lane's program, one executor launch on the whole GPU
    ln = head["dominant"]
    durs = [sum(ctx.run_once(ln["mid"], ln["batch"], ln["x"], ln["y"], 0, True)) for _ in range(3)]
    info = ctx.program_info(ln["mid"], ln["batch"])
    fl, by = sum(s[2] for s in info), sum(s[3] for s in info)
    t = statistics.median(durs) * 1e-9
    tensor = fl / max(by, 1) > peak_burst * 1e12 / (hbm * 1e9)
    ach = fl / t / 1e12 if tensor else by / t / 1e9
    peak = peak_burst if tensor else hbm
    roof = {"bound": "tensor" if tensor else "hbm", "achieved": round(ach, 2), "peak": peak,
            "unit": "TFLOP/s" if tensor else "GB/s", "frac": round(ach / peak, 4), "traffic": None,
            "kernel": f"gl_executor, one launch: {ln['model']} b={ln['batch']} on 148 SMs",
            "launch_us": round(t * 1e6, 1), "algorithmic_flop": fl, "algorithmic_bytes": by,
            "peak_source": f"{peak_src} (MEASURED_PEAKS.json, burst)"}
    sat, tot, dev, wall = aggregate(dist, head["sat"], head["tot"], head["dev_s"], head["wall"])
    if rank != 0:
        ctx.close()
        return None
    line = {
        "metric": METRIC, "value": round(sat / dev, 2), "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(1000 * dev / a.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"cfg4 {a.scenario} (paper game: 6 LeNet-5 + 1 ResNet-50 per app request, P:787) "
                               f"on 1-GPU gpu-let plans, mode {a.mode}" if a.scenario == "game" else
                               f"cfg4 {a.scenario}, mode {a.mode}",
                   "rate_multiplier": round(head["rate_multiplier"], 4), "rates_req_s": head["rates"],
                   "slo_us": slo, "gpulets": head["gpulets"], "lanes": head["lanes"],
                   "requests_per_step": tot / (a.steps * world), "slo_satisfied_frac": round(sat / max(tot, 1), 4),
                   "l2_flush": "none: inputs resident; the six models' weights (~0.58 GB) exceed L2 across steps",
                   "parallelism": f"dp{world} (independent replicas of the 1-GPU plan)"},
        "gpu_launches": len(head["gpulets"]) + 3,
        "wall_req_per_s": round(tot / wall, 2),
        "gpulet_tensor_frac": head["gpulet_tensor_frac"],
        "roofline": roof, "clocks": head["clocks"], "e2e": head["e2e"],
    }
    line.update(extra)
    if not a.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline_sample()
    ctx.close()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="gpulet+int", choices=["gpulet", "gpulet+int", "sbp"])
    ap.add_argument("--scenario", default="game")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--headline-only", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("GL_BENCH_WATCHDOG_S", "1200")), exit=True)
    global VERBOSE
    VERBOSE = a.verbose
    world, rank, local = dist_env()
    if a.impl == "reference":
        line = reference_arm(a, world, rank)
    else:
        dist = init_dist(world, "nccl")
        line = our_arm(a, world, rank, local, dist)
    if line is not None and rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
