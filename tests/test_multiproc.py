"""N > 1 host logic on CPU with gloo, world size 2: the bench's cross-rank
reduction (sum of requests, max of times) and per-rank independent serving of
the same 1-GPU plan (weak scaling), driven through the oracle DES as the fake
GPU backend."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import des, sched
    from tests.test_oracle_sched import W2, prof_from
    from tools.dist_agg import aggregate
    P = prof_from([W2])
    slo = [108_668]
    plan = sched.schedule(P, slo, [700], 1, "gpulet")          # identical 1-GPU plan on every rank
    sim = des.plan_to_sim(plan, P.names)
    arr = {0: des.arrivals_poisson(500, 2_000_000, seed=100 + rank)}   # each rank: own stream, ~70 % load
    st = des.simulate(sim, P, slo, arr)[0]
    ok = st["served"] - st["late"]
    dev_s = 2.0 + 0.1 * rank
    res = aggregate(dist, ok, st["arrivals"], dev_s, dev_s + 0.5)
    q.put((rank, ok, st["arrivals"], res))
    dist.destroy_process_group()


def test_weak_scaling_aggregation_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    sat = sum(o[1] for o in out)
    tot = sum(o[2] for o in out)
    for _r, _ok, _n, res in out:
        assert res[0] == pytest.approx(sat) and res[1] == pytest.approx(tot)
        assert res[2] == pytest.approx(2.1) and res[3] == pytest.approx(2.6)   # max over ranks
    # independent streams: both ranks served most of their load within SLO
    assert sat / tot > 0.9


def _bench_worker(rank, world, port, q):
    """bench.py's own control path at world size 2 (gloo): cross-rank sums /
    maxima and the rate search, which every rank must end identically."""
    import types
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from tests.test_bench_host import FakeServer
    s = bench.allsum(dist, [1.0 + rank, 10.0])
    m = bench.allmax(dist, [0.5 + rank, 3.0 - rank])
    srv = FakeServer(cap=1.1 + 0.2 * rank)     # rank 1 could take more: the summed violations decide
    orig = srv.plan

    def plan(scen, mode, w, x):
        srv._x = x
        return orig(scen, mode, w, x)
    srv.plan = plan
    a = types.SimpleNamespace(probes=10, probe_window=0.01)
    best, probes = bench.search(srv, dist, rank, world, "game", "gpulet", a, 4.0, e2e=False)
    q.put((rank, s, m, best, [p["x"] for p in probes]))
    dist.destroy_process_group()


def test_bench_control_path_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + os.getpid() % 1000
    ps = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _r, s, m, best, xs in out:
        assert s == [3.0, 20.0] and m == [1.5, 3.0]
    # both ranks took the same decisions and agree on the maximum rate
    assert out[0][3] == out[1][3] and out[0][4] == out[1][4]
    assert out[0][3] <= 1.3 and out[0][3] > 1.0
