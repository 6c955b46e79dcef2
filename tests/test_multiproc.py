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
