"""Scheduler-only sweeps on the measured B200 profile.

The paper's schedulability experiment (Fig. success-case): every
model of the five takes a rate in {0, 200, 400, 600} req/s, all-zero excluded
-> 4^5 - 1 = 1,023 scenarios; count how many each scheduler returns
Schedulable.  Its ideal comparison (Fig. ideal_1023): gpulet+int
schedules 18 fewer than the exhaustive ideal (1.8 % of 1,023) on 4 GPUs.

Here every decision is one gl_schedule_files call on the measured B200 files
(profiles/profile_b200.csv, coeffs_b200.json): the profile envelope, the SLOs
(rule or Table constants) and the B200 rate scaling of the paper's rates
(C4.3) are native; a seeded sample of the decisions is replayed through the
oracle (oracle/workload.py + oracle/sched.py) and must be byte-identical.
Modes: SBP on whole GPUs and on 50:50 gpu-lets (Fig. success-case), gpulet,
gpulet+int, and the exhaustive ideal (Fig. ideal_1023); then the maximum
schedulable rate of the five scenarios per mode, normalised to SBP and to the
ideal (Fig. ideal_macrobenchmark).

    python tools/sched_sweep.py [--gpus 1,4] [--modes sbp,sbp50,gpulet,gpulet+int,ideal]
                                [--with-bert] [--slo-mode rule|table] [--json profiles/sched_sweep_b200.json]
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
    ap.add_argument("--modes", default="sbp,sbp50,gpulet,gpulet+int,ideal")
    ap.add_argument("--with-bert", action="store_true", help="6 models (4^6 - 1 = 4,095 scenarios)")
    ap.add_argument("--slo-mode", default="rule", choices=["rule", "table"])
    ap.add_argument("--oracle-sample", type=int, default=40, help="decisions replayed through oracle/")
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    from paper_2109_01611_b200 import gpulet

    prof, coeffs = common.PROFILE_CSV, common.COEFFS_JSON

    def decide(workload):
        """gl_schedule_files: the profile, SLOs and B200 rate scaling are all native (C4)."""
        head, _dump, ok, text = gpulet.schedule_files(prof, coeffs, dict(workload, slo_mode=a.slo_mode))
        return head, ok, text

    nm = 6 if a.with_bert else 5
    names = list(common.MODELS[:nm])
    scen = scenarios(nm)
    head0, _, _ = decide({"rates": [0] * 6})
    out = {"scenarios": len(scen), "levels_req_s_paper": LEVELS, "models": names, "slo_mode": a.slo_mode,
           "slo_us": head0["slo_us"][:nm], "coeffs": common.load_coeffs(),
           "paper": {"ideal_minus_gpulet_int": 18, "of": 1023, "gpus": 4, "cite": "P:927",
                     "success_case": "SBP without vs with 50:50 partitioning, Fig. success-case P:262-270"},
           "results": {}}
    decided = []
    for N in [int(v) for v in a.gpus.split(",")]:
        for mode in a.modes.split(","):
            t0 = time.perf_counter()
            ok = 0
            flags = []
            for r in scen:
                wl = {"base_rates": list(r) + [0] * (6 - nm), "num_gpus": N, "mode": mode}
                _h, sch, _t = decide(wl)
                ok += sch
                flags.append(sch)
                decided.append(wl)
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
    # throughput", and Fig. ideal_macrobenchmark: rates
    # normalised to the ideal's), per scenario, GPU count and mode
    cap = {}
    for sc in ("game", "traffic", "equal", "long-only", "short-skew"):
        for N in (1, 2, 4, 8):
            for mode in ("sbp", "sbp50", "gpulet", "gpulet+int", "ideal"):
                if mode == "ideal" and N > 4:
                    continue

                def ok(x):
                    return decide({"scenario": sc, "x": x, "num_gpus": N, "mode": mode})[1]
                lo, hi = 0.0, 0.25
                while ok(hi) and hi < 1e4:
                    lo, hi = hi, hi * 2
                for _ in range(30):
                    mid = (lo + hi) / 2
                    lo, hi = (mid, hi) if ok(mid) else (lo, mid)
                rates = decide({"scenario": sc, "x": lo, "num_gpus": N, "mode": mode})[0]["rates"]
                cap[f"{sc}@{N}/{mode}"] = {"x": round(lo, 4), "model_req_s": sum(rates) if lo > 0 else 0}
        for N in (1, 2, 4, 8):
            b = cap[f"{sc}@{N}/sbp"]["model_req_s"]
            idl = cap.get(f"{sc}@{N}/ideal", {}).get("model_req_s")
            for mode in ("sbp50", "gpulet", "gpulet+int"):
                g = cap[f"{sc}@{N}/{mode}"]["model_req_s"]
                cap[f"{sc}@{N}/{mode}"]["vs_sbp"] = round(g / b, 3) if b else None
                if idl:
                    cap[f"{sc}@{N}/{mode}"]["vs_ideal"] = round(g / idl, 3)
    out["max_schedulable_rate"] = cap
    ratios = [v["vs_ideal"] for k, v in cap.items() if k.endswith("/gpulet+int") and v.get("vs_ideal") is not None
              and "@4/" in k]
    out["gpulet_int_vs_ideal_rate_at_4"] = {"mean": round(sum(ratios) / len(ratios), 4) if ratios else None,
                                            "min": min(ratios) if ratios else None,
                                            "paper": "92.3 % mean, traffic lowest at 87.7 % (P:939-940)"}
    out["paper_max_rate"] = {"cite": "P:833-852 (4 x 2080 Ti)", "gpulet_vs_sbp": "+106.0 %",
                             "gpulet_int_vs_sbp": "+102.6 %"}
    for k, v in cap.items():
        print(f"{k:28s} {v}", flush=True)
    # oracle replay of a seeded sample (byte-identical outputs: header + plan dump)
    from oracle import workload as owl
    with open(prof) as f:
        ptxt = f.read()
    with open(coeffs) as f:
        ctxt = f.read()
    rnd = random.Random(11)
    sample = rnd.sample(decided, min(a.oracle_sample, len(decided)))
    same, t_or, t_nat = 0, 0.0, 0.0
    for wl in sample:
        t0 = time.perf_counter()
        _h, sch, text = decide(wl)
        t_nat += time.perf_counter() - t0
        t0 = time.perf_counter()
        ref, rok = owl.schedule_files(ptxt, ctxt, json.dumps(dict(wl, slo_mode=a.slo_mode)))
        t_or += time.perf_counter() - t0
        same += (ref == text and rok == sch)
    out["oracle_replay"] = {"sample": len(sample), "identical": same,
                            "oracle_ms_per_decision": round(1e3 * t_or / max(1, len(sample)), 3),
                            "native_ms_per_decision_incl_file_parse": round(1e3 * t_nat / max(1, len(sample)), 3)}
    print(f"oracle replay: {same}/{len(sample)} identical", flush=True)
    for v in out["results"].values():
        if isinstance(v, dict):
            v.pop("_flags", None)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in ("results", "max_schedulable_rate")}))
    print(json.dumps(out["results"]))


if __name__ == "__main__":
    main()
