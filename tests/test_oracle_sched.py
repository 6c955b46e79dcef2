"""Pins for oracle/sched.py (C2), oracle/profiles.py (C4) and oracle/des.py (C5).

Pinned against: SPEC.md worked examples (S:80, S:81, S:100-112, S:170, S:228-247,
S:309-310), SURVEY.md §8(c) C2.13 golden examples W1-W3 (hand-derived),
the SLO-rule invariant b_sat(100) = 32, invariants after every
step, brute force on tiny instances (C2.10), and the
soundness replay through the DES.
"""
import json
import math
import random

import pytest

from oracle import des, profiles, sched
from oracle.sched import GRID, Profile, Scheduler, knee


def prof_from(fns, l2=None, mem=None):
    lat = [[[fn(b, p) for p in GRID] for b in range(1, 33)] for fn in fns]
    return Profile([f"m{i}" for i in range(len(fns))], lat, l2, mem)


def W2(b, p):
    return math.ceil(1000 + 1000 * b * 100 / min(p, 60))


def WB(b, p):
    return math.ceil(500 + 100 * b * 100 / min(p, 40))


def lanes_of(plan):
    return [json.loads(l) for l in plan.dump.splitlines()[:-1]]


# ---- C2.2 / SPEC S:80-81 -------------------------------------------------------
def test_max_feasible_batch_spec_examples():
    P = prof_from([lambda b, p: 5000 * b])       # L(b,100) = 5 b ms
    S = Scheduler(P, [130_000], None, "gpulet")
    assert S.b_sat(0, 100) == 13                 # 2*5b <= 130 -> b = 13 (dense grid)
    S2 = Scheduler(P, [4_000], None, "gpulet")   # SLO < L(1,p)
    assert S2.b_sat(0, 100) is None


def test_slo_rule_gives_batch_32():
    """SLO = 2 L(32,100) => b_sat(m,100) = 32 for any monotone profile."""
    rnd = random.Random(3)
    for _ in range(50):
        a, c = rnd.randint(1, 5000), rnd.randint(1, 3000)
        raw = [[a + c * b * 100 // p + rnd.randint(0, 200) for p in GRID] for b in range(1, 33)]
        env = profiles.envelope(raw)
        P = Profile(["x"], [env])
        S = Scheduler(P, [profiles.slo_rule(env)], None, "gpulet")
        assert S.b_sat(0, 100) == 32


def test_envelope_monotone_idempotent_realizable():
    rnd = random.Random(4)
    raw = [[rnd.randint(100, 10000) for _ in GRID] for _ in range(32)]
    env = profiles.envelope(raw)
    assert profiles.envelope(env) == env
    for b in range(32):
        for g in range(6):
            assert env[b][g] <= raw[b][g]
            if b + 1 < 32:
                assert env[b][g] <= env[b + 1][g]
            if g + 1 < 6:
                assert env[b][g] >= env[b][g + 1]
            # realisable: equals some raw value at b' >= b, p' <= p
            assert any(env[b][g] == raw[bb][gg] for bb in range(b, 32) for gg in range(g + 1))


# ---- C2.4 knee -------------------------------------------------------------------
def test_knee_W1():
    k = sched.curvatures([100, 200, 240, 260, 270, 275])
    assert [round(k[p], 4) for p in (40, 50, 60, 80)] == [0.3237, 1.9907, 2.0603, 0.2858]
    assert knee([100, 200, 240, 260, 270, 275]) == 60
    k2 = sched.curvatures([0, 150, 260, 300, 320, 330])
    assert [round(k2[p], 3) for p in (40, 50, 60, 80)] == [-0.359, 1.519, 2.826, 0.462]
    assert knee([0, 150, 260, 300, 320, 330]) == 60
    assert knee([100, 200, 250, 300, 400, 500]) == 100      # linear: no knee
    assert knee([0] * 6) is None


def test_knee_scale_invariant_and_analytic():
    """Knee invariant under uniform rate scaling and, for the closed form
    L = beta + alpha b 100/p, equal to the argmax of the same curvature."""
    rnd = random.Random(5)
    for _ in range(100):
        r = sorted(rnd.randint(1, 1000) for _ in range(6))
        s = rnd.randint(2, 9)
        assert knee(r) == knee([x * s for x in r])
        k = sched.curvatures(r)
        best = knee(r)
        if best != 100:
            assert k[best] == max(v for p, v in k.items() if v > 1e-9)


# ---- C2.5 p_req + W2 ---------------------------------------------------------------
def test_W2_curve_and_plans():
    P = prof_from([W2])
    slo = [2 * W2(32, 100)]
    assert slo == [108_668]
    S = Scheduler(P, slo, None, "gpulet")
    assert [S.b_sat(0, p) for p in GRID] == [10, 21, 26, 32, 32, 32]
    assert [P.L(0, S.b_sat(0, p), p) for p in GRID] == [51_000, 53_500, 53_000, 54_334, 54_334, 54_334]
    assert S.curve(0) == [196, 392, 490, 588, 588, 588]
    assert round(sched.curvatures(S.curve(0))[60], 4) == 5.4263
    assert S.p_eff(0) == 60
    assert S.p_req(0, 300) == 40 and S.p_req(0, 5000) == 100 and S.p_req(0, 0) == 20

    plan = sched.schedule(P, slo, [300], 1, "gpulet")
    assert plan.ok
    gl = lanes_of(plan)
    assert [(g["slot"], g["size"], g["sm"]) for g in gl] == [(0, 40, 60), (1, 60, 88)]   # exact SM shares (DESIGN R15)
    assert gl[0]["lanes"] == [{"model": "m0", "rate": 300, "batch": 21, "exec_us": 53_500, "F": 1000}]
    assert gl[1]["lanes"] == []

    plan = sched.schedule(P, slo, [700], 1, "gpulet")
    gl = lanes_of(plan)
    assert plan.ok
    assert (gl[0]["size"], gl[0]["lanes"][0]["rate"], gl[0]["lanes"][0]["batch"], gl[0]["lanes"][0]["exec_us"]) == (60, 588, 32, 54_334)
    assert (gl[1]["size"], gl[1]["lanes"][0]["rate"], gl[1]["lanes"][0]["batch"], gl[1]["lanes"][0]["exec_us"]) == (40, 112, 21, 53_500)

    assert not sched.schedule(P, slo, [2000], 1, "gpulet").ok
    assert sched.schedule(P, slo, [1900], 2, "gpulet").ok   # 2 x (588 + 392) = 1960


def test_W3_merge_path():
    P = prof_from([W2, WB])
    slo = [2 * W2(32, 100), 2 * WB(32, 100)]
    assert slo[1] == 17_000
    S = Scheduler(P, slo, None, "gpulet")
    assert S.curve(1) == [1882, 3764, 3764, 3764, 3764, 3764] and S.p_eff(1) == 40
    plan = sched.schedule(P, slo, [200, 100], 1, "gpulet")
    gl = lanes_of(plan)
    assert plan.ok
    assert gl[0] == {"gpu": 0, "slot": 0, "size": 40, "sm": 60, "D_us": 8500, "lanes": [
        {"model": "m0", "rate": 200, "batch": 2, "exec_us": 6000, "F": 1000},
        {"model": "m1", "rate": 100, "batch": 1, "exec_us": 750, "F": 1000}]}
    assert gl[1]["size"] == 60 and gl[1]["lanes"] == []
    # A at 300: b_A = 3, e_A = 8,500 -> sum e > D, no merge; B keeps slot 1
    gl = lanes_of(sched.schedule(P, slo, [300, 100], 1, "gpulet"))
    assert [len(g["lanes"]) for g in gl] == [1, 1] and gl[1]["lanes"][0]["model"] == "m1"


# ---- merge predicate, SPEC S:237-247 ------------------------------------------------
def test_temporally_sharable_examples():
    # A: duty 40 ms exec 20 ms (SLO 95); B: duty 40 exec 15 (SLO 130): flat latency tables
    P = prof_from([lambda b, p: 20_000 if b <= 2 else 40_000, lambda b, p: 15_000 if b <= 2 else 40_000])
    S = Scheduler(P, [95_000, 130_000], None, "gpulet")
    g = sched.Gpulet(0, 0, 100)
    ev = S.eval_lanes(g, None, lanes=[sched.Lane(0, 50), sched.Lane(1, 50)])
    assert ev is not None and ev[0] == 40_000 and sum(r[2] for r in ev[1]) == 35_000
    # LeNet-like 5 ms SLO lane with a 90 ms exec lane: not sharable
    P2 = prof_from([lambda b, p: 1_000, lambda b, p: 90_000])
    S2 = Scheduler(P2, [5_000, 200_000], None, "gpulet")
    assert S2.eval_lanes(g, None, lanes=[sched.Lane(0, 10), sched.Lane(1, 1)]) is None


def test_factor_arithmetic_S170():
    c = (0.2, 0.1, 0.5, 0.3, 1.0)
    l2 = [[[0.5] * 6 for _ in range(6)]]
    mem = [[[0.4] * 6 for _ in range(6)]]
    P = Profile(["x"], [[[100_000] * 6 for _ in range(32)]], l2, mem)
    S = Scheduler(P, [10**9], c, "gpulet+int")
    assert S.factor(0, 4, 50, (0.5, 0.4)) == 1470           # 1.47
    assert S.leff(0, 4, 50, 1470) == 147_000                 # overhead 47 ms on 100 ms
    S0 = Scheduler(P, [10**9], (0, 0, 0, 0, 0.9), "gpulet+int")
    assert S0.factor(0, 4, 50, (0.5, 0.4)) == 1000           # raw 0.9 clamps to 1.0
    assert S.factor(0, 4, 50, None) == 1000                   # no partner


# ---- best fit / split / revert, SPEC S:228-230, S:309-310 ----------------------------
def test_best_fit_split_revert():
    P = prof_from([W2])
    S = Scheduler(P, [108_668], None, "gpulet")
    S.fixed = False
    S.remain = [sched.Gpulet(0, 0, 40), sched.Gpulet(0, 1, 60), sched.Gpulet(1, 0, 100)]
    S.alloc = []
    r = S.find_best_fit(0, 50, 100)
    assert r == 100 and S.alloc[0].size == 60                 # p_ideal 50 -> best fit 60
    S.remain, S.alloc = [sched.Gpulet(0, 0, 100)], []
    S.find_best_fit(0, 40, 100)
    assert S.alloc[0].size == 40 and [g.size for g in S.remain] == [60]   # split, take 40
    # split then revert is the identity
    g = sched.Gpulet(0, 0, 100)
    S.remain = [g]
    t, s = S._split(g, 40)
    assert (t.size, s.size) == (40, 60)
    S._unsplit(g, t, s)
    assert S.remain == [g]


# ---- invariants over random instances -------------------------------------------------
def _random_instance(rnd, M):
    fns, l2, mem = [], [], []
    for _ in range(M):
        a, c, sat = rnd.randint(200, 5000), rnd.randint(50, 3000), rnd.choice([40, 50, 60, 80, 100])
        fns.append(lambda b, p, a=a, c=c, sat=sat: a + (c * b * 100 + min(p, sat) - 1) // min(p, sat))
        l2.append([[rnd.random() * 0.8 for _ in GRID] for _ in range(6)])
        mem.append([[rnd.random() * 0.8 for _ in GRID] for _ in range(6)])
    P = prof_from(fns, l2, mem)
    slo = [2 * P.L(m, 32, 100) for m in range(M)]
    return P, slo


def _check_invariants(plan, rates, S_mode, P, slo, N):
    per_gpu = {}
    for g in lanes_of(plan):
        per_gpu.setdefault(g["gpu"], []).append(g["size"])
    for gpu, sizes in per_gpu.items():
        assert sum(sizes) == 100 and len(sizes) <= 2
    if plan.ok:
        tot = {}
        for g in lanes_of(plan):
            for ln in g["lanes"]:
                tot[ln["model"]] = tot.get(ln["model"], 0) + ln["rate"]
                assert ln["batch"] <= 32 and ln["F"] >= 1000
            if g["lanes"]:
                assert sum(ln["exec_us"] for ln in g["lanes"]) <= g["D_us"]
                ms = [ln["model"] for ln in g["lanes"]]
                assert len(set(ms)) == len(ms)
        for m, r in enumerate(rates):
            assert tot.get(P.names[m], 0) == r


@pytest.mark.parametrize("mode", ["gpulet", "gpulet+int", "sbp"])
def test_invariants_random(mode):
    rnd = random.Random(11)
    c = (0.1, 0.15, 0.2, 0.25, 1.0)
    for _ in range(60):
        M, N = rnd.randint(1, 4), rnd.randint(1, 3)
        P, slo = _random_instance(rnd, M)
        S = Scheduler(P, slo, c, "gpulet")
        rates = [rnd.choice([0, rnd.randint(1, 3 * max(1, S.cap(m, 100)))]) for m in range(M)]
        if not any(rates):
            continue
        plan = sched.schedule(P, slo, rates, N, mode, c)
        _check_invariants(plan, rates, mode, P, slo, N)
        # determinism
        assert sched.schedule(P, slo, rates, N, mode, c).dump == plan.dump


def test_elastic_implies_brute_force():
    """elastic Schedulable => brute force Schedulable (N = 1, M <= 2, small rates)."""
    rnd = random.Random(12)
    gaps = 0
    for _ in range(25):
        M = rnd.randint(1, 2)
        P, slo = _random_instance(rnd, M)
        # scale latencies so that tiny rates matter
        P.lat = [[[x * 400 for x in row] for row in lat] for lat in P.lat]
        slo = [2 * P.L(m, 32, 100) for m in range(M)]
        rates = [rnd.randint(1, 12) for _ in range(M)]
        for mode in ("gpulet", "gpulet+int"):
            c = (0.1, 0.1, 0.2, 0.2, 1.0)
            e = sched.schedule(P, slo, rates, 1, mode, c).ok
            bf = sched.brute_force(P, slo, rates, mode, c)
            assert not (e and not bf)
            gaps += (bf and not e)
    assert gaps <= 25


def _worked_profile(names):
    fns = {"W2": W2, "WB": WB}
    return prof_from([fns[n] for n in names]), None


def test_sbp_and_ideal_worked_examples():
    """Hand-derived SBP / SBP-on-50:50 / ideal plans (tests/golden/sched_sbp_ideal_worked.json,
    each with its derivation): the oracle reproduces every dump byte for byte."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "sched_sbp_ideal_worked.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        P, _ = _worked_profile(case["profile"])
        P.names = ["A", "B"][:len(case["profile"])]
        if case["mode"] == "ideal":
            plan = sched.ideal(P, case["slo"], case["rates"], case["gpus"], "gpulet+int", (0, 0, 0, 0, 0))
        else:
            plan = sched.schedule(P, case["slo"], case["rates"], case["gpus"], case["mode"])
        assert plan.dump == "\n".join(case["dump"]) + "\n", case["name"]


def test_ideal_dominates_on_tiny():
    """Any instance Alg. 1 schedules with its split at a layout of the ideal's grid is
    also schedulable by the ideal (it tries that layout); on random tiny instances the
    ideal's verdict is at least the elastic one whenever the elastic plan's layout is
    one of {100}, {20,80}, {40,60}, {50,50}."""
    rnd = random.Random(13)
    checked = 0
    for _ in range(40):
        M, N = rnd.randint(1, 3), rnd.randint(1, 2)
        P, slo = _random_instance(rnd, M)
        S = Scheduler(P, slo, None, "gpulet")
        rates = [rnd.randint(1, 2 * max(1, S.cap(m, 100))) for m in range(M)]
        plan = sched.schedule(P, slo, rates, N, "gpulet")
        if not plan.ok:
            continue
        sizes = {}
        for g in plan.gpulets:
            sizes.setdefault(g.gpu, []).append(g.size)
        if all(tuple(sorted(v)) in {(100,), (20, 80), (40, 60), (50, 50)} for v in sizes.values()):
            assert sched.ideal(P, slo, rates, N, "gpulet+int", (0, 0, 0, 0, 0)).ok
            checked += 1
    assert checked >= 5


def test_layout_count():
    from itertools import combinations_with_replacement
    assert len(list(combinations_with_replacement(range(4), 4))) == 35
    assert len(list(combinations_with_replacement(range(4), 8))) == 165


def test_scenarios():
    assert 4 ** 5 - 1 == 1023
    from itertools import product
    suite = [r for r in product([0, 100], repeat=3) if any(r)]
    assert len(suite) == 7
    assert profiles.app_rates("game", 10) == (60, 0, 10, 0, 0, 0)
    assert profiles.app_rates("traffic", 10) == (0, 10, 0, 10, 10, 0)


# ---- C5 DES ----------------------------------------------------------------------------
def test_poisson_and_determinism():
    a = des.arrivals_poisson(100, 100_000_000, seed=7)
    assert abs(len(a) - 10_000) < 3 * 100                      # mean within 3 sigma
    assert a == des.arrivals_poisson(100, 100_000_000, seed=7)
    assert a != des.arrivals_poisson(100, 100_000_000, seed=8)


@pytest.mark.parametrize("mode", ["gpulet", "gpulet+int", "sbp"])
def test_soundness_replay(mode):
    """Every Schedulable plan replays with 0 violations under deterministic
    arrivals at exactly the plan rates."""
    rnd = random.Random(21)
    c = (0.05, 0.05, 0.1, 0.1, 1.0)
    checked = 0
    for _ in range(40):
        M, N = rnd.randint(1, 3), rnd.randint(1, 2)
        P, slo = _random_instance(rnd, M)
        S = Scheduler(P, slo, c, "gpulet")
        rates = [rnd.randint(1, max(2, S.cap(m, 100))) for m in range(M)]
        plan = sched.schedule(P, slo, rates, N, mode, c)
        if not plan.ok:
            continue
        sim = des.plan_to_sim(plan, P.names)
        dur = 20 * max(slo)
        arr = {}
        for gsize, D, ls in sim:
            pass
        # per-lane deterministic arrivals: each model's arrivals at its total rate
        arr = {m: des.arrivals_deterministic(rates[m], dur) for m in range(M) if rates[m]}
        st = des.simulate(sim, P, slo, arr)
        for m, s in st.items():
            assert s["violations"] == 0, (mode, m, s["late"], s["dropped"], plan.dump)
        checked += 1
    assert checked >= 5


def test_interference_aware_batch_is_maximal():
    """Reading R13: with a partner the batch is the largest
    b <= b_sat whose interference-inflated latency still fits the duty-cycle
    rule 2 Leff <= SLO; a zero-slack b_sat (SLO = 2 L(32)) must shrink."""
    P = prof_from([W2])
    slo = [2 * P.L(0, 32, 100)]
    S = sched.Scheduler(P, slo, (0.0, 0.0, 0.0, 0.0, 1.2), "gpulet+int")
    A = (0.5, 0.5)
    for p in (40, 60, 100):
        b0 = S.b_sat(0, p)
        b = S.b_int(0, p, A)
        assert b is not None and b < b0
        assert 2 * S.leff(0, b, p, S.factor(0, b, p, A)) <= slo[0]
        assert 2 * S.leff(0, b + 1, p, S.factor(0, b + 1, p, A)) > slo[0]
        assert S.b_int(0, p, None) == b0          # no partner: solo b_sat
