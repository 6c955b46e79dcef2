"""File-driven scheduler boundary (SURVEY §8(b) gl_schedule on SPEC-format files):
native gl_profile_load / gl_workload_rates / gl_schedule_files vs the oracle
(oracle/workload.py + oracle/sched.py).  Outputs — SLOs, rates, plan dumps with
their header — must be byte-identical, and the two sides
must fail on the same malformed inputs with the same error kind.  CPU only."""
import json
import math
import os

import pytest

from oracle import workload as W
from paper_2109_01611_b200 import gpulet

pytestmark = pytest.mark.skipif(not os.path.exists(gpulet.LIB_PATH), reason="libgpulet.so not built")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILE = os.path.join(ROOT, "profiles", "profile_b200.csv")
COEFFS = os.path.join(ROOT, "profiles", "coeffs_b200.json")
SCENARIOS = ("game", "traffic", "equal", "mix6", "long-only", "short-skew")
KIND = {"parse": -9, "data": -10, "arg": -1}


def _read(p):
    with open(p) as f:
        return f.read()


def _native(profile, coeffs, workload):
    return gpulet.schedule_files(profile, coeffs, workload)[3]


def _oracle(profile, coeffs, workload):
    return W.schedule_files(_read(profile), None if coeffs is None else _read(coeffs), json.dumps(workload))[0]


def test_profile_tables_identical():
    lat, l2, mem, sm = gpulet.profile_load(PROFILE)
    ref = W.parse_profile(_read(PROFILE))
    assert lat.tolist() == ref["lat"]
    assert l2.tolist() == ref["l2"] and mem.tolist() == ref["mem"]
    assert sm.tolist() == ref["sm"]


@pytest.mark.parametrize("slo_mode", ["rule", "table"])
def test_rates_identical(slo_mode):
    lat, *_ = gpulet.profile_load(PROFILE)
    ref_lat = W.parse_profile(_read(PROFILE))["lat"]
    ref_slo = W.slos(ref_lat, slo_mode)
    for scen in SCENARIOS:
        for x in (0.0, 0.01, 0.37, 1.0, 1.5, 2.75, 13.0 / 7.0, 40.0):
            for n in (1, 2, 4, 8):
                slo, rates = gpulet.workload_rates(lat, scen, x, n, slo_mode)
                assert slo == ref_slo
                assert rates == W.scenario_rates(scen, ref_slo, x, n)[0], (scen, x, n)


@pytest.mark.parametrize("slo_mode", ["rule", "table"])
@pytest.mark.parametrize("mode", ["gpulet", "gpulet+int", "sbp", "sbp50"])
def test_bench_scenarios_identical(mode, slo_mode):
    """Every bench scenario at N in {1,2,4,8}, on a ladder of multipliers that
    crosses each scenario's schedulability edge."""
    for scen in SCENARIOS:
        for n in (1, 2, 4, 8):
            for x in (0.05, 0.3, 0.9, 1.7, 3.1, 6.0):
                wl = {"scenario": scen, "x": x, "num_gpus": n, "mode": mode, "slo_mode": slo_mode}
                assert _native(PROFILE, COEFFS, wl) == _oracle(PROFILE, COEFFS, wl), wl


def test_ideal_models_and_rates_forms_identical():
    for n in (1, 2, 4):
        wl = {"scenario": "equal", "x": 0.8, "num_gpus": n, "mode": "ideal"}
        assert _native(PROFILE, COEFFS, wl) == _oracle(PROFILE, COEFFS, wl)
    for base in ([200, 0, 400, 600, 0, 0], [600, 600, 600, 600, 600, 600], [0, 200, 0, 0, 0, 400]):
        for mode in ("gpulet", "sbp", "gpulet+int", "sbp50"):
            wl = {"base_rates": base, "x": 1.0, "num_gpus": 4, "mode": mode}
            assert _native(PROFILE, COEFFS, wl) == _oracle(PROFILE, COEFFS, wl)
    wl = {"rates": [300, 20, 40, 10, 5, 3], "num_gpus": 2, "mode": "gpulet+int"}
    assert _native(PROFILE, COEFFS, wl) == _oracle(PROFILE, COEFFS, wl)
    wl = {"models": [{"name": "resnet50", "rate": 700, "slo_ms": 95}, {"name": "vgg16", "rate": 150, "slo_ms": 12.5}],
          "num_gpus": 1, "mode": "gpulet", "slo_mode": "table"}
    assert _native(PROFILE, None, wl) == _oracle(PROFILE, None, wl)


def test_truncated_rates_not_schedulable():
    """A multiplier so small that ResNet-50's game rate floors to 0 is not a
    game workload any more: NotSchedulable without a plan."""
    wl = {"scenario": "game", "x": 0.0001, "mode": "gpulet"}
    head, dump, ok, text = gpulet.schedule_files(PROFILE, COEFFS, wl)
    assert not ok and head["rates"][2] == 0 and head["rates"][0] > 0
    assert json.loads(dump)["reason"] == "rate_truncated"
    assert text == _oracle(PROFILE, COEFFS, wl)


def _synthetic_csv(path, fn=lambda m, b, p: 100 * (m + 1) + math.ceil(1000 * b / p), ms=False, drop=None, extra=None,
                   sm=True):
    rows = ["model,batch,partition_pct" + (",sm_count" if sm else "") + (",latency_ms" if ms else ",latency_us")
            + ",l2_util,mem_bw_util"]
    for m, name in enumerate(W.NAMES):
        for b in range(1, 33):
            for gi, p in enumerate(W.GRID):
                if drop == (name, b, p):
                    continue
                v = fn(m, b, p)
                lat = f"{v / 1000}" if ms else str(v)
                st = f"{0.1 * (gi + 1) / 6:.6f},{0.05 * (m + 1) / 6:.6f}" if b in W.STAT_B else ","
                rows.append(f"{name},{b},{p}" + (f",{W.SM_DEFAULT[gi]}" if sm else "") + f",{lat},{st}")
    if extra:
        rows.append(extra)
    with open(path, "w") as f:
        f.write("\n".join(rows) + "\n")
    return str(path)


def _kind_native(fn):
    with pytest.raises(gpulet.GpuletError) as e:
        fn()
    return e.value.code


def _kind_oracle(fn):
    with pytest.raises(W.WorkloadError) as e:
        fn()
    return KIND[e.value.kind]


def test_latency_ms_and_noisy_profiles_identical(tmp_path):
    # SPEC's unit (ms, decimals) and a non-monotone (noisy) table that only the envelope repairs
    p = _synthetic_csv(tmp_path / "a.csv", fn=lambda m, b, p: 1000 + 37 * b * (m + 1) + (b * 7919 + p) % 113, ms=True)
    for mode in ("gpulet", "gpulet+int", "sbp"):
        for scen in ("equal", "game", "traffic"):
            wl = {"scenario": scen, "x": 1.0, "mode": mode, "num_gpus": 2}
            assert _native(p, COEFFS, wl) == _oracle(p, COEFFS, wl)
    lat, *_ = gpulet.profile_load(p)
    assert lat.tolist() == W.parse_profile(_read(p))["lat"]
    # strict mode (SPEC S:41-42 / S:58): the noisy table is a data error on both sides
    wl = {"scenario": "equal", "envelope": False}
    assert _kind_native(lambda: gpulet.schedule_files(p, None, wl)) == -10
    assert _kind_oracle(lambda: W.schedule_files(_read(p), None, json.dumps(wl))) == -10


@pytest.mark.parametrize("case", ["missing", "duplicate", "unknown_model", "off_grid", "bad_batch", "util_range",
                                  "malformed_latency", "field_count", "zero_latency", "sm_mismatch"])
def test_profile_errors_same_kind(tmp_path, case):
    base = dict(fn=lambda m, b, p: 100 + b)
    extra = {
        "duplicate": "lenet5,1,20,30,7,,",
        "unknown_model": "alexnet,1,20,30,7,,",
        "off_grid": "lenet5,1,30,30,7,,",
        "bad_batch": "lenet5,33,20,30,7,,",
        "util_range": "lenet5,1,20,30,7,1.5,0.1",
        "malformed_latency": "lenet5,1,20,30,7x,,",
        "field_count": "lenet5,1,20,30",
        "zero_latency": "lenet5,1,20,30,0,,",
        "sm_mismatch": "lenet5,1,20,31,7,,",
    }
    if case == "missing":
        p = _synthetic_csv(tmp_path / "e.csv", drop=("vgg16", 17, 60), **base)
    else:
        p = _synthetic_csv(tmp_path / "e.csv", **base)
        # the extra row duplicates (lenet5, 1, 20) unless it is malformed first: drop the real one
        text = _read(p).replace("lenet5,1,20,30,101,", "lenet5,1,20,30,XX,", 1) if case != "duplicate" else _read(p)
        lines = [ln for ln in text.splitlines() if "XX" not in ln] + [extra[case]]
        with open(p, "w") as f:
            f.write("\n".join(lines) + "\n")
    n = _kind_native(lambda: gpulet.profile_load(p))
    o = _kind_oracle(lambda: W.parse_profile(_read(p)))
    assert n == o, (case, n, o)


def test_workload_json_errors():
    for bad in ('{"scenario": "game"', '{"scenario": "nope"}', '{"scenario": "game", "rates": [1,2,3,4,5,6]}',
                '{"rates": [1, 2]}', '{"scenario": "game", "mode": "fifo"}', '[1, 2]'):
        code = _kind_native(lambda: gpulet.schedule_files(PROFILE, COEFFS, bad))
        assert code in (-9, -1), bad
    with pytest.raises(gpulet.GpuletError):
        gpulet.schedule_files(PROFILE, None, {"scenario": "game", "mode": "gpulet+int"})   # needs coefficients


@pytest.mark.parametrize("slo_mode", ["rule", "table"])
@pytest.mark.parametrize("mode", ["gpulet", "gpulet+int", "sbp"])
def test_traffic_chain_identical(mode, slo_mode):
    """Scenario "traffic-chain" (F3, DESIGN R28): stage-split SLOs (header app_slo_us),
    app-SLO-scaled rates and the plan, byte-identical, with and without a hand-off
    reservation; gl_workload_rates agrees with the oracle (hand-off 0)."""
    for n in (1, 2, 4):
        for x in (0.01, 0.2, 0.9, 2.5):
            for h in (0, 130):
                wl = {"scenario": "traffic-chain", "x": x, "num_gpus": n, "mode": mode, "slo_mode": slo_mode,
                      "handoff_us": h}
                assert _native(PROFILE, COEFFS, wl) == _oracle(PROFILE, COEFFS, wl), wl
    lat, *_ = gpulet.profile_load(PROFILE)
    ref_lat = W.parse_profile(_read(PROFILE))["lat"]
    slo, rates = gpulet.workload_rates(lat, "traffic-chain", 0.7, 2, slo_mode)
    ref_slo, ref_rates, _s_app = W.chain_workload(ref_lat, slo_mode, 0.7, 2)
    assert slo == ref_slo and rates == ref_rates
