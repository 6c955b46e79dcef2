"""Scheduler-only sweeps on the measured B200 profile.

The paper's schedulability experiment (Fig. success-case): every
model of the five takes a rate in {0, 200, 400, 600} req/s, all-zero excluded
-> 4^5 - 1 = 1,023 scenarios; count how many each scheduler returns
Schedulable.  Its ideal comparison (Fig. ideal_1023): gpulet+int
schedules 18 fewer than the exhaustive ideal (1.8 % of 1,023) on 4 GPUs.

Here the rates are scaled to B200 by SLO_paper / SLO_B200 per model (C4.3),
the profile / SLOs / interference coefficients are the measured B200 ones
(profiles/profile_b200.csv, coeffs_b200.json), and the native scheduler
(libgpulet gl_schedule, CPU code) decides; a seeded sample of the decisions
is replayed through the oracle (oracle/sched.py) and must be byte-identical.

    python tools/sched_sweep.py [--gpus 1,4] [--modes sbp,gpulet,gpulet+int,ideal]
                                [--with-bert] [--json profiles/sched_sweep_b200.json]
"""
import argparse
import itertools
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from tools import common  # noqa: E402

LEVELS = (0, 200, 400, 600)


def scenarios(n_models):
    return [r for r in itertools.product(LEVELS, repeat=n_models) if any(r)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", default="1,4")
    ap.add_argument("--modes", default="sbp,gpulet,gpulet+int,ideal")
    ap.add_argument("--with-bert", action="store_true", help="6 models (4^6 - 1 = 4,095 scenarios)")
    ap.add_argument("--oracle-sample", type=int, default=40, help="decisions replayed through oracle/sched.py")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    from paper_2109_01611_b200 import gpulet

    lat, l2, mem = common.read_profile_csv(common.PROFILE_CSV)
    lat_env = [common.envelope(lat[m]) for m in range(len(common.MODELS))]
    slo = common.slos_from(lat_env)
    coeffs = common.load_coeffs()
    nm = 6 if a.with_bert else 5
    names = list(common.MODELS[:nm])
    scale = []
    for m in names:
        ref = m if m in common.PAPER_SLO_MS else "resnet50"
        scale.append(common.PAPER_SLO_MS[ref] * 1000.0 / slo[common.MODELS.index(ref)])
    L, L2, ME, S = lat_env[:nm], l2[:nm], mem[:nm], slo[:nm]
    scen = scenarios(nm)
    out = {"scenarios": len(scen), "levels_req_s_paper": LEVELS, "models": names,
           "b200_rate_scale": [round(s, 3) for s in scale], "slo_us": S, "coeffs": list(coeffs),
           "paper": {"ideal_minus_gpulet_int": 18, "of": 1023, "gpus": 4, "cite": "P:927"}, "results": {}}
    decided = []
    for N in [int(v) for v in a.gpus.split(",")]:
        for mode in a.modes.split(","):
            t0 = time.perf_counter()
            ok = 0
            flags = []
            for r in scen:
                rates = [int(v * s) for v, s in zip(r, scale)]
                _dump, sch = gpulet.schedule(names, L, L2, ME, S, rates, N, mode, coeffs)
                ok += sch
                flags.append(sch)
                decided.append((N, mode, rates))
            dt = time.perf_counter() - t0
            out["results"][f"{mode}@{N}"] = {"schedulable": ok, "of": len(scen),
                                             "native_ms_per_decision": round(1e3 * dt / len(scen), 4)}
            out["results"][f"{mode}@{N}"]["_flags"] = flags
            print(f"N={N} {mode:11s} schedulable {ok:5d} / {len(scen)}  ({1e3 * dt / len(scen):.3f} ms/decision)",
                  flush=True)
    for N in [int(v) for v in a.gpus.split(",")]:
        if f"ideal@{N}" in out["results"] and f"gpulet+int@{N}" in out["results"]:
            i, g = out["results"][f"ideal@{N}"], out["results"][f"gpulet+int@{N}"]
            out["results"][f"ideal_minus_gpulet_int@{N}"] = i["schedulable"] - g["schedulable"]
            # Alg. 1 is a heuristic inside the ideal's search space: a scenario it
            # schedules must also be schedulable by the ideal
            out["results"][f"gpulet_int_not_ideal@{N}"] = sum(
                1 for x, y in zip(g["_flags"], i["_flags"]) if x and not y)
    # scheduler-level maximum rates (the paper's Fig. "maximum achievable
    # throughput", before serving validation): per scenario, GPU
    # count and mode, the largest rate multiplier the scheduler accepts
    cap = {}
    full_l2, full_mem = l2, mem
    for scen in ("game", "traffic", "equal", "long-only", "short-skew"):
        for N in (1, 2, 4, 8):
            for mode in ("sbp", "gpulet", "gpulet+int"):
                def ok(x):
                    rates = common.scenario_rates(scen, slo, x)
                    return gpulet.schedule(common.MODELS, lat_env, full_l2, full_mem, slo, [r * N for r in rates],
                                           N, mode, coeffs)[1] and sum(rates) > 0
                lo, hi = 0.0, 0.25
                while ok(hi) and hi < 1e4:
                    lo, hi = hi, hi * 2
                for _ in range(30):
                    mid = (lo + hi) / 2
                    lo, hi = (mid, hi) if ok(mid) else (lo, mid)
                rates = common.scenario_rates(scen, slo, lo)
                cap[f"{scen}@{N}/{mode}"] = {"x": round(lo, 4), "model_req_s": sum(rates) * N}
        for N in (1, 2, 4, 8):
            b = cap[f"{scen}@{N}/sbp"]["model_req_s"]
            for mode in ("gpulet", "gpulet+int"):
                g = cap[f"{scen}@{N}/{mode}"]["model_req_s"]
                cap[f"{scen}@{N}/{mode}"]["vs_sbp"] = round(g / b, 3) if b else None
    out["max_schedulable_rate"] = cap
    out["paper_max_rate"] = {"cite": "P:833-852 (4 x 2080 Ti)", "gpulet_vs_sbp": "+106.0 %",
                             "gpulet_int_vs_sbp": "+102.6 %"}
    for k, v in cap.items():
        if k.endswith("gpulet+int") or k.endswith("gpulet"):
            print(f"{k:28s} {v}", flush=True)
    # oracle replay of a seeded sample (byte-identical plan dumps)
    from oracle import sched as osched
    P = osched.Profile(names, L, L2, ME)
    rnd = random.Random(11)
    sample = rnd.sample(decided, min(a.oracle_sample, len(decided)))
    same, t_or = 0, 0.0
    for N, mode, rates in sample:
        dump, sch = gpulet.schedule(names, L, L2, ME, S, rates, N, mode, coeffs)
        t0 = time.perf_counter()
        ref = osched.ideal(P, S, rates, N, "gpulet+int", coeffs) if mode == "ideal" else \
            osched.schedule(P, S, rates, N, mode, coeffs)
        t_or += time.perf_counter() - t0
        same += (ref.dump == dump and ref.ok == sch)
    out["oracle_replay"] = {"sample": len(sample), "identical": same,
                            "oracle_ms_per_decision": round(1e3 * t_or / max(1, len(sample)), 3)}
    print(f"oracle replay: {same}/{len(sample)} identical", flush=True)
    for v in out["results"].values():
        if isinstance(v, dict):
            v.pop("_flags", None)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "results"}))
    print(json.dumps(out["results"]))


if __name__ == "__main__":
    main()
