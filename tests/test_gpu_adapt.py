"""Live gpu-let reorganisation on a B200 (PAPER.md P:672-676:
a changed plan re-partitions the GPU): a plan whose gpu-let sizes change is
deployed by destroying the old executors and creating the new ones (green
contexts, sized programs), traffic served before and after completes, and a
plan that keeps the sizes only re-plans the lanes (no executor restart)."""
import json
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan(sizes, batches=(8, 4)):
    gls = [{"gpu": 0, "slot": 0, "size": sizes[0], "sm": 0, "D_us": 60,
            "lanes": [{"model": "lenet5", "rate": 2000, "batch": batches[0], "exec_us": 30, "F": 1000}]},
           {"gpu": 0, "slot": 1, "size": sizes[1], "sm": 0, "D_us": 2000,
            "lanes": [{"model": "resnet50", "rate": 200, "batch": batches[1], "exec_us": 900, "F": 1000}]}]
    return "\n".join(json.dumps(g) for g in gls) + "\n" + json.dumps({"verdict": "Forced"})


def test_live_reorganisation_keeps_serving():
    import bench
    from paper_2109_01611_b200 import gpulet
    ctx = gpulet.Context(1)
    srv = bench.Server(ctx, 0, False)
    try:
        slo = [10**7] * 6
        my = srv.setup(_plan((20, 80)), 0)
        assert srv.made_nsm == [30, 118]
        t, m = bench.poisson_trace(my, 0.2, 11)
        assert (ctx.serve(srv.lanes, 6, t, m, slo) >= 0).all()
        t0 = time.perf_counter()
        my = srv.setup(_plan((50, 50)), 0, reuse=True)
        reorg_s = time.perf_counter() - t0
        assert srv.reorganised and srv.made_nsm == [74, 74]
        assert reorg_s < 5.0, reorg_s
        t, m = bench.poisson_trace(my, 0.2, 12)
        lat = ctx.serve(srv.lanes, 6, t, m, slo)
        assert (lat >= 0).all() and len(lat) > 100
        gids = list(srv.made)
        my = srv.setup(_plan((50, 50), batches=(16, 2)), 0, reuse=True)   # same sizes: lanes only
        assert not srv.reorganised and srv.made == gids
        assert [ln["batch"] for ln in srv.lanes] == [16, 2]
        t, m = bench.poisson_trace(my, 0.2, 13)
        assert (ctx.serve(srv.lanes, 6, t, m, slo) >= 0).all()
    finally:
        srv.teardown()
        ctx.close()
