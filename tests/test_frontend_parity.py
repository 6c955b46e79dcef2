"""Frontend routing + dispatch + drop decisions (SURVEY §8(a) a5/a6, §8(c) C2.11,
DESIGN R26): libgpulet's gl_serve_sim — the dispatch rule gl_serve runs, driven
by a virtual clock against FIFO gpu-lets — must produce exactly the oracle DES's
batch sequence (lane, dispatch time, size, first request) and per-request
latencies on seeded traces.  Plus hand-traced DES pins for every condition of
the rule.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import des
from oracle import sched as osched
from oracle import workload as W
from paper_2109_01611_b200 import gpulet

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILE = os.path.join(ROOT, "profiles", "profile_b200.csv")
COEFFS = os.path.join(ROOT, "profiles", "coeffs_b200.json")
native_lib = pytest.mark.skipif(not os.path.exists(gpulet.LIB_PATH), reason="libgpulet.so not built")


class Flat:
    """Profile with L(k, p) = lat[k - 1] on every p (hand-traced pins)."""

    def __init__(self, lat):
        self.lat = lat

    def L(self, m, k, p):
        return self.lat[k - 1]


def trace_of(pairs):
    return [(t, m) for t, m in pairs]


# ---- hand-traced pins of the DES (C2.11 + R26) --------------------------------------------
def test_batch_formed():
    """b = 2, long duty cycle: the second arrival (t = 10) completes the batch; end = 10 + 100."""
    lat, log = des.simulate_trace([(100, 10**6, [(0, 1, 2, 1000)])], Flat([100] * 32), [10_000],
                                  trace_of([(0, 0), (10, 0)]))
    assert log == [(0, 10, 2, 0)] and lat == [110, 100]


def test_duty_cycle_timeout():
    """b = 4, D = 1000: a lone request at t = 100 waits for the window (opened at 0) to pass."""
    lat, log = des.simulate_trace([(100, 1000, [(0, 1, 4, 1000)])], Flat([100] * 32), [10_000],
                                  trace_of([(100, 0)]))
    assert log == [(0, 1000, 1, 0)] and lat == [1000]


def test_deadline_guard_uses_the_batch_it_would_send():
    """SLO 500, Leff(1) = 100, Leff(2) = 200: after the second arrival the lane must go by
    0 + 500 - Leff(2) = 300 (R26), and both requests finish at exactly their SLO."""
    lat, log = des.simulate_trace([(100, 10**6, [(0, 1, 4, 1000)])], Flat([100, 200] + [300] * 30), [500],
                                  trace_of([(0, 0), (50, 0)]))
    assert log == [(0, 300, 2, 0)] and lat == [500, 450]


def test_hopeless_requests_dropped():
    """SLO below Leff(1): nothing can be served, every request dropped (-1)."""
    lat, log = des.simulate_trace([(100, 1000, [(0, 1, 4, 1000)])], Flat([600] * 32), [500],
                                  trace_of([(0, 0), (5, 0), (7, 0)]))
    assert log == [] and lat == [-1, -1, -1]


def test_fifo_gpulet_and_smooth_wrr():
    """Two lanes of model 0 on one gpu-let with weights 2:1 -> A, B, A; batches of 1 queue
    behind each other on the gpu-let (start = max(t, free))."""
    lat, log = des.simulate_trace([(100, 10**6, [(0, 2, 1, 1000)]), (0, 10**6, [])], Flat([100] * 32), [10**6],
                                  trace_of([(0, 0), (0, 0), (0, 0)]))
    # a single gpu-let hosting one lane: 3 batches at t = 0 back to back
    assert log == [(0, 0, 1, 0), (0, 0, 1, 1), (0, 0, 1, 2)] and lat == [100, 200, 300]
    plan = [(50, 10**6, [(0, 2, 1, 1000), (1, 5, 1, 1000)]), (50, 10**6, [(0, 1, 1, 1000)])]
    lat, log = des.simulate_trace(plan, Flat([100] * 32), [10**6, 10**6],
                                  trace_of([(0, 0), (1, 0), (2, 0), (3, 1)]))
    assert [row[0] for row in log] == [0, 2, 0, 1]          # model 0: lanes 0, 2, 0 (weights 2:1); model 1: lane 1
    assert lat == [100, 100, 198, 297]                      # lanes 0 and 1 share gpu-let 0's FIFO


def test_model_without_lane_dropped():
    lat, log = des.simulate_trace([(100, 10, [(0, 1, 1, 1000)])], Flat([5] * 32), [100, 100],
                                  trace_of([(0, 1), (3, 0)]))
    assert lat == [-1, 5] and log == [(0, 3, 1, 1)]


class PerModel:
    """Profile with L(k, p) = lat[m] for every k and p (hand-traced chain pins)."""

    def __init__(self, lat):
        self.lat = lat

    def L(self, m, k, p):
        return self.lat[m]


CHAIN_PLAN = [(100, 10**6, [(0, 1, 1, 1000)]), (50, 1000, [(1, 1, 2, 1000)]), (50, 10**6, [(2, 1, 1, 1000)])]


def test_chain_hand_traced():
    """F3 two-stage chain (DESIGN R28): detector m0 (L 100, b 1) spawns one m1 (L 50,
    b 2, D 1000) and one m2 (L 30, b 1) request per completed request, 7 µs later,
    each keeping its root's arrival.  t=0: m0 batch -> end 100, spawns 2,3 at 107;
    t=10: m0 batch starts when the gpu-let frees at 100 -> end 200, spawns 4,5 at 207;
    t=107: 3 dispatches alone (b 1) -> 137; 2 waits (b 2, window 0 + D 1000, deadline
    0 + 5000 - 50); t=207: 4 completes m1's batch [2, 4] -> 257, 5 -> 237."""
    lat, log, parent, model = des.simulate_trace(CHAIN_PLAN, PerModel([100, 50, 30]), [1000, 5000, 5000],
                                                 [(0, 0), (10, 0)], spawn={0: [1, 2]}, handoff_us=7)
    assert lat == [100, 190, 257, 137, 247, 227]
    assert parent == [-1, -1, 0, 0, 1, 1] and model == [0, 0, 1, 2, 1, 2]
    assert log == [(0, 0, 1, 0), (0, 10, 1, 1), (2, 107, 1, 3), (1, 207, 2, 2), (2, 207, 1, 5)]
    assert des.app_latencies(lat, parent, 2) == [257, 247]


def test_chain_drops_propagate():
    """A hopeless second-stage request is dropped ((107 - 0) + 30 > 120) and fails its
    application; a dropped first-stage request spawns nothing."""
    lat, log, parent, model = des.simulate_trace(CHAIN_PLAN, PerModel([100, 50, 30]), [1000, 5000, 120],
                                                 [(0, 0), (10, 0)], spawn={0: [1, 2]}, handoff_us=7)
    assert lat[3] == -1 and des.app_latencies(lat, parent, 2)[0] == -1
    lat, log, parent, model = des.simulate_trace(CHAIN_PLAN, PerModel([100, 50, 30]), [150, 5000, 5000],
                                                 [(0, 0), (10, 0)], spawn={0: [1, 2]}, handoff_us=7)
    # request 1 would end at 200 > 10 + 150: dropped at its dispatch (t = 10: 0 + 100 > 150? no -> sent);
    # it is late (190 > 150) but still spawns; only a drop stops the chain
    assert lat[:2] == [100, 190] and len(lat) == 6
    lat, log, parent, model = des.simulate_trace(CHAIN_PLAN, PerModel([100, 50, 30]), [90, 5000, 5000],
                                                 [(0, 0), (10, 0)], spawn={0: [1, 2]}, handoff_us=7)
    assert lat == [-1, -1] and parent == [-1, -1] and des.app_latencies(lat, parent, 2) == [-1, -1]


def test_chain_empty_spawn_is_plain():
    plan = [(100, 1000, [(0, 1, 4, 1000)])]
    tr = [(0, 0), (5, 0), (3000, 0)]
    lat0, log0 = des.simulate_trace(plan, Flat([100] * 32), [10_000], tr)
    lat1, log1, parent, model = des.simulate_trace(plan, Flat([100] * 32), [10_000], tr, spawn={})
    assert (lat0, log0) == (lat1, log1) and parent == [-1] * 3 and model == [0, 0, 0]


def test_guard_margin():
    """R29: a lone request (b = 4, long duty cycle, L = 100, SLO 500) is sent by the
    deadline guard at t = 500 - 100 = 400 (ends at the SLO); with a 50 µs margin at
    t = 350 (ends 50 µs inside it)."""
    lat, log = des.simulate_trace([(100, 10**6, [(0, 1, 4, 1000)])], Flat([100] * 32), [500], [(0, 0)])
    assert lat == [500] and log == [(0, 400, 1, 0)]
    lat, log = des.simulate_trace([(100, 10**6, [(0, 1, 4, 1000, 50)])], Flat([100] * 32), [500], [(0, 0)])
    assert lat == [450] and log == [(0, 350, 1, 0)]


# ---- native gl_serve_sim == oracle DES ------------------------------------------------------------
def _lanes_from_plan(dump, prof_lat):
    plan, lanes = [], []
    for gi, line in enumerate(ln for ln in dump.splitlines() if '"gpu"' in ln):
        d = json.loads(line)
        if not d["lanes"]:
            continue
        ls = []
        for ln in d["lanes"]:
            m = W.NAMES.index(ln["model"])
            g = W.GRID.index(d["size"])
            leff = [(prof_lat[m][k - 1][g] * ln["F"] + 999) // 1000 for k in range(1, 33)]
            ls.append((m, ln["rate"], ln["batch"], ln["F"]))
            lanes.append(dict(gpulet=100 + len(plan), model_slot=m, batch=ln["batch"], duty_us=d["D_us"],
                              weight=ln["rate"], drop_us=leff[0], leff_us=leff))
        plan.append((d["size"], d["D_us"], ls))
    return plan, lanes


def _poisson(rates, secs, seed):
    ts, ms = [], []
    for m, r in enumerate(rates):
        if r <= 0:
            continue
        rng = np.random.Generator(np.random.PCG64(seed * 131 + m))
        t = np.cumsum(-np.log(1.0 - rng.random(int(r * secs * 1.3) + 20)) / r * 1e6)
        t = t[t < secs * 1e6].astype(np.int64)
        ts.append(t)
        ms.append(np.full(len(t), m, np.int32))
    t, m = np.concatenate(ts), np.concatenate(ms)
    o = np.argsort(t, kind="stable")
    return t[o], m[o]


@native_lib
@pytest.mark.parametrize("scen,mode,x,n", [("game", "gpulet", 1.0, 1), ("game", "gpulet", 3.0, 1),
                                           ("traffic", "gpulet", 0.4, 1), ("equal", "gpulet+int", 0.7, 4),
                                           ("mix6", "sbp", 0.2, 8), ("short-skew", "gpulet", 1.5, 2)])
@pytest.mark.parametrize("load", [0.8, 1.3])
def test_serve_sim_equals_des(scen, mode, x, n, load):
    """Plans from the measured profile (n GPUs: every GPU's gpu-lets in one replay);
    Poisson traffic at 0.8x and 1.3x (overload: the deadline guard and the drop rule
    fire) of the planned rates."""
    prof = W.parse_profile(open(PROFILE).read())
    for _ in range(12):   # halve x until schedulable on one GPU
        head, dump, ok, _ = gpulet.schedule_files(PROFILE, COEFFS, {"scenario": scen, "x": x, "mode": mode, "num_gpus": n})
        if ok:
            break
        x /= 2
    assert ok
    plan, lanes = _lanes_from_plan(dump, prof["lat"])
    if load > 1:   # overload case: every lane with a jitter reserve (R29), same on both sides
        mg = [(3 * i + 1) % 7 for i in range(len(lanes))]     # lane i of the plan order, both sides
        it = iter(mg)
        plan = [(sz, D, [lt + (next(it),) for lt in ls]) for sz, D, ls in plan]
        lanes = [dict(ln, margin_us=g) for ln, g in zip(lanes, mg)]
    rates = [r * load for r in head["rates"]]
    t, m = _poisson(rates, 0.2, seed=int(100 * x) + int(10 * load))
    lat_n, log_n = gpulet.serve_sim(lanes, 6, t, m, head["slo_us"])
    lat_o, log_o = des.simulate_trace(plan, osched.Profile(W.NAMES, prof["lat"]), head["slo_us"],
                                      list(zip(t.tolist(), m.tolist())))
    assert log_n == log_o
    assert lat_n.tolist() == lat_o
    assert len(log_o) > 10


@native_lib
def test_serve_sim_edge_cases():
    lanes = [dict(gpulet=0, model_slot=0, batch=2, duty_us=100, weight=1, drop_us=10, leff_us=[10] * 32)]
    lat, log = gpulet.serve_sim(lanes, 2, [], [], [50, 50])
    assert lat.tolist() == [] and log == []
    lat, log = gpulet.serve_sim(lanes, 2, [0, 0, 0, 5], [0, 1, 0, 0], [50, 50])
    lat_o, log_o = des.simulate_trace([(100, 100, [(0, 1, 2, 1000)])], Flat([10] * 32), [50, 50],
                                      [(0, 0), (0, 1), (0, 0), (5, 0)])
    assert lat.tolist() == lat_o and log == log_o
    with pytest.raises(gpulet.GpuletError):
        gpulet.serve_sim([dict(lanes[0], leff_us=None)], 2, [0], [0], [50, 50])
    with pytest.raises(gpulet.GpuletError):
        gpulet.serve_sim(lanes, 2, [5, 0], [0, 0], [50, 50])


# ---- application chains (F3, DESIGN R28): native gl_serve_sim_chain == oracle DES ----------
@native_lib
def test_serve_sim_chain_hand_traced():
    lanes = []
    for gi, (size, D, ls) in enumerate(CHAIN_PLAN):
        for (m, rate, b, F) in ls:
            lanes.append(dict(gpulet=gi, model_slot=m, batch=b, duty_us=D, weight=rate, drop_us=[100, 50, 30][m],
                              leff_us=[[100, 50, 30][m]] * 32))
    lat, log, parent, model = gpulet.serve_sim_chain(lanes, 3, [0, 10], [0, 0], [1000, 5000, 5000], {0: [1, 2]}, 7)
    assert lat.tolist() == [100, 190, 257, 137, 247, 227]
    assert parent.tolist() == [-1, -1, 0, 0, 1, 1] and model.tolist() == [0, 0, 1, 2, 1, 2]
    assert log == [(0, 0, 1, 0), (0, 10, 1, 1), (2, 107, 1, 3), (1, 207, 2, 2), (2, 207, 1, 5)]
    lat, log, parent, model = gpulet.serve_sim_chain(lanes, 3, [0, 10], [0, 0], [90, 5000, 5000], {0: [1, 2]}, 7)
    assert lat.tolist() == [-1, -1] and parent.tolist() == [-1, -1]


@native_lib
@pytest.mark.parametrize("load", [0.7, 1.4])
@pytest.mark.parametrize("handoff", [0, 130])
def test_serve_sim_chain_equals_des_traffic(load, handoff):
    """`traffic` as a two-stage chain on the measured profile: the stage-split SLOs and
    rates of scenario "traffic-chain" (R28) planned by gl_schedule_files, Poisson SSD
    app arrivals; every SSD completion spawns one GoogLeNet and one VGG-16 request."""
    prof = W.parse_profile(open(PROFILE).read())
    lat_env = prof["lat"]
    ssd, goo, vgg = W.NAMES.index("ssd_mobilenet_v1"), W.NAMES.index("googlenet"), W.NAMES.index("vgg16")
    x = 1.0
    for _ in range(12):
        head, dump, ok, _ = gpulet.schedule_files(PROFILE, COEFFS, {"scenario": "traffic-chain", "x": x,
                                                                    "handoff_us": handoff, "mode": "gpulet", "num_gpus": 2})
        if ok:
            break
        x /= 2
    assert ok
    s_app = head["app_slo_us"]
    assert head["slo_us"][ssd] + head["slo_us"][goo] + handoff == s_app
    plan, lanes = _lanes_from_plan(dump, lat_env)
    slo = list(head["slo_us"])
    slo[goo] = slo[vgg] = s_app                    # from the application's arrival
    t, m = _poisson([0, 0, 0, head["rates"][ssd] * load, 0, 0], 0.3, seed=7 + handoff)
    lat_n, log_n, par_n, mdl_n = gpulet.serve_sim_chain(lanes, 6, t, m, slo, {ssd: [goo, vgg]}, handoff)
    lat_o, log_o, par_o, mdl_o = des.simulate_trace(plan, osched.Profile(W.NAMES, lat_env), slo,
                                                    list(zip(t.tolist(), m.tolist())), spawn={ssd: [goo, vgg]},
                                                    handoff_us=handoff)
    assert log_n == log_o and lat_n.tolist() == lat_o
    assert par_n.tolist() == par_o and mdl_n.tolist() == mdl_o
    assert len(lat_o) == len(t) + 2 * sum(1 for x in lat_o[:len(t)] if x >= 0)
    assert len(log_o) > 10
