"""Diagnostic: LeNet-5 SLO misses in the game headline vs the deadline-guard
margin (DESIGN R29).  For the game plan at multiplier x, serve Poisson windows
with margin_us in {0, 2, 4, 8, 12} on every lane and print the violation
fraction, late vs dropped LeNet requests and latency percentiles; plus the
host-observed service-time distribution of LeNet b1 batches on its gpu-let."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    import bench
    from paper_2109_01611_b200 import gpulet
    from tools import common
    xs = [float(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1.0,2.5").split(",")]
    ctx = gpulet.Context(1)
    srv = bench.Server(ctx, 0, False)
    out = []
    for x in xs:
        rates, dump, ok = srv.plan("game", "gpulet", 1, x)
        my = srv.setup(dump, 0)
        # host-observed LeNet b1 service time on its gpu-let
        ln = next(l for l in srv.lanes if l["model"] == "lenet5")
        ts = []
        for i in range(400):
            t0 = time.perf_counter()
            ctx.wait(ctx.submit_batch(ln["gpulet"], ln["model_id"], ln["x"], ln["y"], 1))
            ts.append((time.perf_counter() - t0) * 1e6)
        ts = np.array(ts[50:])
        svc = {"p50": float(np.percentile(ts, 50)), "p99": float(np.percentile(ts, 99)),
               "p999": float(np.percentile(ts, 99.9)), "max": float(ts.max())}
        print("x", x, "lenet b1 host service us", json.dumps(svc), flush=True)
        base = [dict(l) for l in srv.lanes]
        for mg in (0, 2, 4, 8, 12):
            srv.lanes = [dict(l, margin_us=mg) for l in base]
            res = []
            for r in range(3):
                t, m = bench.poisson_trace(my, 0.5, 7000 + r)
                lat = ctx.serve(srv.lanes, len(common.MODELS), t, m, srv.slo)
                sel = m == 0
                ll = lat[sel]
                slo = srv.slo[0]
                ok_l = ll[ll >= 0]
                res.append({"viol_all": float(((lat < 0) | (lat > np.asarray(srv.slo)[m])).mean()),
                            "lenet_late": int((ll > slo).sum()), "lenet_drop": int((ll < 0).sum()),
                            "lenet_n": int(sel.sum()), "p50": float(np.percentile(ok_l, 50)),
                            "p99": float(np.percentile(ok_l, 99)), "p999": float(np.percentile(ok_l, 99.9))})
            row = {"x": x, "margin_us": mg, "runs": res}
            out.append(row)
            print(json.dumps(row), flush=True)
        srv.teardown()
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(out, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
