"""Host logic of bench.py (no GPU): the rate search (R19, median of three runs,
P:823), the serving-window roofline (R24) and the Poisson trace."""
import types

import numpy as np

import bench


class FakeServer:
    """Violations jump above 1 % once x exceeds `cap`; records the probes."""

    slo_mode = "rule"

    def __init__(self, cap):
        self.cap, self.lanes, self.calls = cap, [], []
        self.gpu = 0

    def max_sched_x(self, scen, mode, world):
        return 4.0

    def plan(self, scen, mode, world, x):
        return [100, 0, 10, 0, 0, 0], "dump", True

    def setup(self, dump, rank):
        return [100, 0, 10, 0, 0, 0]

    def teardown(self):
        pass

    def window(self, my, secs, seed, e2e=False):
        x = self._x
        self.calls.append(x)
        arr = 10000
        cap = getattr(self, "cap_timed", self.cap) if secs == getattr(self, "timed_secs", None) else self.cap
        viol = 5 if x <= cap else 500
        return {"arrivals": arr, "viol": viol, "per": {}, "sat": arr - viol, "dev_s": secs, "wall_s": secs,
                "lanes": []}


def test_search_bisects_to_the_cap():
    a = types.SimpleNamespace(probes=12, probe_window=0.01)
    srv = FakeServer(cap=1.37)
    orig = srv.plan

    def plan(scen, mode, world, x):
        srv._x = x
        return orig(scen, mode, world, x)
    srv.plan = plan
    best, probes = bench.search(srv, None, 0, 1, "game", "gpulet", a, 4.0, e2e=False)
    assert best is not None and best <= 1.37 and best > 1.37 * 0.97
    assert all(len(srv.calls[i:i + 3]) == 3 for i in range(0, len(srv.calls), 3))   # 3 runs per probe
    assert probes[0]["viol_frac"] > 0.01


def test_roofline_serving_picks_busiest_lane_and_bound():
    util = [{"model": "lenet5", "gpulet_pct": 20, "sm": 24, "planned_batch": 24, "batches": 10, "requests": 30,
             "busy_s": 0.001, "mean_batch": 3.0, "mean_batch_us": 100.0, "tflops": 0.05, "tensor_frac": 0.0002,
             "tensor_peak_tflops": 227.0, "gbs": 3.0, "hbm_frac": 0.0005, "hbm_peak_gbs": 6650.0, "peak_source": "x"},
            {"model": "resnet50", "gpulet_pct": 80, "sm": 124, "planned_batch": 15, "batches": 10, "requests": 100,
             "busy_s": 0.01, "mean_batch": 10.0, "mean_batch_us": 1000.0, "tflops": 80.0, "tensor_frac": 0.068,
             "tensor_peak_tflops": 1173.0, "gbs": 60.0, "hbm_frac": 0.009, "hbm_peak_gbs": 6650.0, "peak_source": "x"}]
    r = bench.roofline_serving(util)
    assert r["bound"] == "tensor" and r["achieved"] == 80.0 and r["peak"] == 1173.0
    assert abs(r["frac"] - 80.0 / 1173.0) < 1e-3
    util[1]["gbs"] = 1e6    # FLOP per byte below the ridge -> HBM-bound
    assert bench.roofline_serving(util)["bound"] == "hbm"
    # the dominant lane is the one that used the most GPU (busy time x SMs), not the busiest clock
    util[1]["gbs"] = 60.0
    util[0]["busy_s"] = 0.02
    assert bench.roofline_serving(util)["kernel"].startswith("gl_executor serving resnet50")


def test_poisson_trace_rates_and_order():
    t, m = bench.poisson_trace([2000, 0, 500, 0, 0, 0], 2.0, 3, lead_us=0)
    assert np.all(np.diff(t) >= 0)
    n0, n2 = int((m == 0).sum()), int((m == 2).sum())
    assert abs(n0 - 4000) < 5 * np.sqrt(4000) and abs(n2 - 1000) < 5 * np.sqrt(1000)
    assert int((m == 1).sum()) == 0


def test_timed_runs_enforce_the_rule():
    """The probes pass at x but the timed windows (a tighter cap) violate: run_mode must
    lower x until every timed run meets <= 1 %, value = the median run."""
    a = types.SimpleNamespace(probes=12, probe_window=0.01, window=0.02, steps=2, warmup=0, repeats=3, retries=6,
                              e2e=False)
    srv = FakeServer(cap=1.37)
    srv.cap_timed, srv.timed_secs = 1.2, 0.02     # the timed windows see a lower capacity than the probes
    orig = srv.plan

    def plan(scen, mode, world, x):
        srv._x = x
        return orig(scen, mode, world, x)
    srv.plan = plan
    r = bench.run_mode(srv, None, 0, 1, "game", "gpulet", a)
    assert r["criterion_met"] and r["x"] <= 1.2
    assert all(v["viol_frac"] <= 0.01 for v in r["repeats"]) and len(r["repeats"]) == 3
    assert len(r["attempts"]) >= 2 and max(r["attempts"][0]["viol_frac"]) > 0.01
