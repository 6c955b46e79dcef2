"""Consolidation curves for two models on one GPU (partial;
PAPER.md P:257-276, Fig. slo-violation: SLO violation of LeNet and VGG-16
when they are consolidated with different resource sharing schemes).

Schemes, on the same kernels and the same Poisson traces:
  temporal   one 100 % gpu-let, both models as lanes of one executor (the
             whole-GPU temporal sharing of SBP): each lane's batch
             is its largest SLO-feasible batch at 100 %, the shared duty cycle
             is the longest of the two lanes' execution times;
  spatial    two gpu-lets, 20 % for LeNet and 80 % for VGG-16 (the paper's
             "MPS(20:80)"): each lane on its own gpu-let with its own duty cycle;
  unconfined the paper's third scheme, concurrent kernels without a static SM
             partition ("MPS(default)"; two persistent executors
             without green contexts, gl_create_gpulets_unconfined): the same two
             lanes on two executors of the primary context whose CTAs the
             hardware places; one executor CTA fills an SM, so each still runs a
             fixed CTA count (20:80, and 50:50 -- no size policy at all).

For rate multipliers x (the models' B200-scaled paper rates times x), the
violation fraction (late + dropped) of each model is measured.

    python tools/consolidate.py [--xs 0.1,0.2,...] [--secs 1.0] [--json profiles/consolidate_b200.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


SCHEMES = ("temporal", "spatial-20:80", "unconfined-20:80", "unconfined-50:50")


def lane(model, rate, batch, exec_us):
    return {"model": model, "rate": int(rate), "batch": int(batch), "exec_us": int(exec_us), "F": 1000}


def b_sat(lat_env, mi, gi, slo_us):
    """Largest batch with 2 L(b, p) <= SLO (R4), or 1."""
    best = 1
    for b in range(1, 33):
        if 2 * lat_env[mi][b - 1][gi] <= slo_us:
            best = b
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="lenet5,vgg16")
    ap.add_argument("--xs", default="0.05,0.1,0.2,0.3,0.4,0.6,0.8,1.0")
    ap.add_argument("--secs", type=float, default=1.0)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    import bench
    from paper_2109_01611_b200 import gpulet
    from tools import common

    ctx = gpulet.Context(1)
    srv = bench.Server(ctx, 0, False)
    lat_env, slo = srv.lat, srv.slo
    small, large = a.models.split(",")
    ms, ml = common.MODELS.index(small), common.MODELS.index(large)
    g100, g20, g80 = common.GRID.index(100), common.GRID.index(20), common.GRID.index(80)
    base = [0] * len(common.MODELS)
    # the paper's 100 req/s per model, scaled to B200 (C4.3, gl_workload_rates' per-model
    # scale: the "long-only" scenario is 100 req/s of ResNet/SSD/VGG/BERT, "short-skew" 100 of LeNet)
    lo = srv.scenario_rates("long-only", 1.0)
    sk = srv.scenario_rates("short-skew", 1.0)
    for m in (ms, ml):
        base[m] = float(lo[m] if lo[m] else sk[m])
    out = {"models": [small, large], "slo_us": [slo[ms], slo[ml]], "base_req_s": [base[ms], base[ml]],
           "secs": a.secs, "cite": "P:257-276", "curves": {k: [] for k in SCHEMES}}
    for x in [float(v) for v in a.xs.split(",")]:
        rates = [int(r * x) for r in base]
        for scheme in SCHEMES:
            if scheme == "temporal":
                bs, bl = b_sat(lat_env, ms, g100, slo[ms]), b_sat(lat_env, ml, g100, slo[ml])
                es, el = lat_env[ms][bs - 1][g100], lat_env[ml][bl - 1][g100]
                d = max(es, el)
                gls = [{"gpu": 0, "slot": 0, "size": 100, "sm": 148, "D_us": int(d),
                        "lanes": [lane(small, rates[ms], bs, es), lane(large, rates[ml], bl, el)]}]
            else:
                ps, pl = (50, 50) if scheme.endswith("50:50") else (20, 80)
                gs, gl_ = common.GRID.index(ps), common.GRID.index(pl)
                bs, bl = b_sat(lat_env, ms, gs, slo[ms]), b_sat(lat_env, ml, gl_, slo[ml])
                es, el = lat_env[ms][bs - 1][gs], lat_env[ml][bl - 1][gl_]
                gls = [{"gpu": 0, "slot": 0, "size": ps, "sm": 0, "D_us": int(es),
                        "lanes": [lane(small, rates[ms], bs, es)]},
                       {"gpu": 0, "slot": 1, "size": pl, "sm": 0, "D_us": int(el),
                        "lanes": [lane(large, rates[ml], bl, el)]}]
            dump = "\n".join(json.dumps(g) for g in gls) + "\n" + json.dumps({"verdict": "Forced"})
            my = srv.setup(dump, 0, unconfined=scheme.startswith("unconfined"))
            smids = [sorted(ctx.gpulet_smids(gid)) for gid in srv.made] if scheme.startswith("unconfined") else None
            w = srv.window(my, a.secs, 900 + int(100 * x))
            srv.teardown()
            per = w["per"]
            row = {"x": x, "rates": [rates[ms], rates[ml]], "batches": [bs, bl],
                   "viol_frac": {m: round(per[m]["viol"] / max(per[m]["arrivals"], 1), 4) for m in (small, large)
                                 if m in per},
                   "p99_us": {m: per[m]["p99_us"] for m in (small, large) if m in per}}
            if smids:
                row["smids"] = smids
            out["curves"][scheme].append(row)
            print(scheme, json.dumps(row), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
