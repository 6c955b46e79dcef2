"""Pins of oracle/workload.py (C4: profile files, SLOs, rates) against what the
paper and arithmetic fix — not against the oracle itself."""
import json
import math

import pytest

from oracle import workload as W


def _csv(fn, ms=False, sm=None):
    rows = ["model,batch,partition_pct,sm_count," + ("latency_ms" if ms else "latency_us") + ",l2_util,mem_bw_util"]
    for m, name in enumerate(W.NAMES):
        for b in range(1, 33):
            for gi, p in enumerate(W.GRID):
                rows.append(f"{name},{b},{p},{(sm or W.SM_DEFAULT)[gi]},{fn(m, b, p)},,")
    return "\n".join(rows) + "\n"


def test_table_slos_are_the_papers():
    """Table tab:ml-models: goo 44, le 5, res 95, ssd 136, vgg 130 ms."""
    slo = W.slos(None, "table")
    assert dict(zip(W.NAMES, slo)) == {"lenet5": 5000, "googlenet": 44000, "resnet50": 95000,
                                       "ssd_mobilenet_v1": 136000, "vgg16": 130000, "bert_base": 95000}


def test_table_mode_rates_are_the_papers_rates():
    """SLO_B200 = SLO_paper -> scale 1: Table tab:particular-scenarios."""
    slo = W.slos(None, "table")
    assert W.scenario_rates("equal", slo)[0] == [50] * 6
    assert W.scenario_rates("long-only", slo)[0] == [0, 0, 100, 100, 100, 100]
    assert W.scenario_rates("short-skew", slo)[0] == [100, 100, 100, 50, 50, 50]
    assert W.scenario_rates("short-skew", slo, 1.0, 4)[0] == [400, 400, 400, 200, 200, 200]


def test_app_compositions_survive_scaling():
    """game = 6 LeNet + 1 ResNet-50 per app request; traffic = SSD + GoogLeNet + VGG-16 1:1:1
     — for any SLOs and multipliers (one scale per application, R23)."""
    slo = [56, 1996, 2784, 2800, 4076, 3626]
    for x in (0.5, 1.0, 2.0, 4.0):
        g = W.scenario_rates("game", slo, x)[0]
        t = W.scenario_rates("traffic", slo, x)[0]
        assert g[1] == g[3] == g[4] == g[5] == 0 and abs(g[0] - 6 * g[2]) <= 6
        assert t[0] == t[2] == t[5] == 0 and t[1] == t[3] == t[4]


def test_rule_mode_hand_computed():
    """L(b,p) = 1000 + 100 b on every p for every model -> L*(32,100) = 4200 µs, SLO = 8400 µs
    (P:764-766 doubling rule).  equal at x = 1: 50 * 95 ms / 8.4 ms = 565.47... -> 565 ResNet-50
    req/s; LeNet 50 * 5 / 8.4 = 29.76 -> 29; BERT uses ResNet-50's scale -> 565."""
    P = W.parse_profile(_csv(lambda m, b, p: 1000 + 100 * b))
    slo = W.slos(P["lat"], "rule")
    assert slo == [8400] * 6
    r = W.scenario_rates("equal", slo)[0]
    assert r == [29, 261, 565, 809, 773, 565]
    assert 50 * 44 / 8.4 == pytest.approx(261.9, abs=0.1) and 50 * 136 / 8.4 == pytest.approx(809.5, abs=0.1)


def test_exact_decimal_latency():
    """0.1 ms is 100 µs exactly (binary 0.1 * 1000 = 100.00000000000001 would ceil to 101);
    0.1001 ms rounds up to 101 µs (C2.1 ceil)."""
    P = W.parse_profile(_csv(lambda m, b, p: "0.1" if b < 32 else "0.1001", ms=True), strict=True)
    assert P["lat"][0][0][0] == 100 and P["lat"][0][31][5] == 101


def test_envelope_is_min_over_dominated_cells():
    """Brute-force definition (C4.1) on a random table; idempotent; monotone."""
    import random
    rng = random.Random(5)
    lat = [[rng.randint(10, 99) for _ in W.GRID] for _ in range(32)]
    env = W.envelope(lat)
    for b in range(32):
        for g in range(6):
            want = min(lat[bb][gg] for bb in range(32) for gg in range(6) if bb >= b and gg <= g)
            assert env[b][g] == want
            assert b == 0 or env[b][g] >= env[b - 1][g]
            assert g == 0 or env[b][g] <= env[b][g - 1]
    assert W.envelope(env) == env


def test_sm_counts_come_from_the_file():
    P = W.parse_profile(_csv(lambda m, b, p: 100 + b, sm=(24, 48, 56, 72, 96, 148)))
    assert P["sm"] == [24, 48, 56, 72, 96, 148]
    P = W.parse_profile(_csv(lambda m, b, p: 100 + b).replace(",30,", ",,", 3).replace("sm_count", "sm_count"))
    assert P["sm"][0] == 30


def test_strict_mode_rejects_non_monotone():
    text = _csv(lambda m, b, p: 100 + b if (m, b, p) != (2, 5, 40) else 10)
    with pytest.raises(W.WorkloadError) as e:
        W.parse_profile(text, strict=True)
    assert e.value.kind == "data"
    W.parse_profile(text)   # the envelope repairs it


def test_truncation_reported():
    text = _csv(lambda m, b, p: 1000 + 100 * b)
    out, ok = W.schedule_files(text, None, json.dumps({"scenario": "game", "x": 0.01}))
    head = json.loads(out.splitlines()[0])
    # ResNet-50: floor(100 * 95000 * 0.01 / 8400) = floor(11.3) = 11 > 0 -> not truncated at 0.01
    assert head["rates"][2] == 11 and ok in (True, False)
    out, ok = W.schedule_files(text, None, json.dumps({"scenario": "game", "x": 0.0008}))
    head, verdict = [json.loads(ln) for ln in out.splitlines()]
    assert head["rates"][2] == 0 and not ok and verdict["reason"] == "rate_truncated"
    assert math.floor(600 * 95000 * 0.0008 / 8400) == head["rates"][0] > 0


def test_traffic_stage_slos_hand_computed():
    """R28 on a hand-made table (L at b = 32, 100 %): SSD 1000, GoogLeNet 500, VGG 3000 µs.
    Rule: s_app = 2 * 3000 (the longest member doubled); s1 = 6000 * 1000 /
    (1000 + 3000) = 1500; the recognisers get 6000 - 1500 - handoff.  Table: 136 ms
    (P:791), s1 = 136000 / 4 = 34000.  Rates: floor(100 * 136000 * x / s_app)."""
    from oracle import workload as W
    lat = [[[1] * 6 for _ in range(32)] for _ in W.NAMES]
    for m, v in (("ssd_mobilenet_v1", 1000), ("googlenet", 500), ("vgg16", 3000)):
        lat[W.NAMES.index(m)][31][5] = v
    assert W.traffic_stage_slos(lat, "rule") == (6000, 1500)
    assert W.traffic_stage_slos(lat, "table") == (136000, 34000)
    slo, rates, s_app = W.chain_workload(lat, "rule", x=0.5, num_gpus=2, handoff_us=100)
    i = W.NAMES.index
    assert s_app == 6000 and slo[i("ssd_mobilenet_v1")] == 1500
    assert slo[i("googlenet")] == slo[i("vgg16")] == 4400
    assert rates[i("ssd_mobilenet_v1")] == rates[i("vgg16")] == (100 * 136000 // 2 // 6000) * 2 == 2266
    assert rates[i("lenet5")] == rates[i("resnet50")] == rates[i("bert_base")] == 0
    import pytest
    with pytest.raises(W.WorkloadError):
        W.traffic_stage_slos(lat, "rule", handoff_us=4500)
