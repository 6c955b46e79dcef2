"""Native scheduler (libgpulet gl_schedule) vs the oracle (oracle/sched.py):
plan dumps must be byte-identical.  CPU only: the
scheduler is host code inside libgpulet.so."""
import math
import random

import pytest

from oracle import sched
from oracle.sched import GRID, Profile
from paper_2109_01611_b200 import gpulet

pytestmark = pytest.mark.skipif(not __import__("os").path.exists(gpulet.LIB_PATH), reason="libgpulet.so not built")


def native(P, slo, rates, N, mode, c=None):
    return gpulet.schedule(P.names, P.lat, P.l2, P.mem, slo, rates, N, mode, c)


def _check(P, slo, rates, N, mode, c=None):
    if mode == "ideal":
        ref = sched.ideal(P, slo, rates, N, "gpulet+int", c)
    else:
        ref = sched.schedule(P, slo, rates, N, mode, c)
    dump, ok = native(P, slo, rates, N, mode, c)
    assert dump == ref.dump, (mode, rates, N)
    assert ok == ref.ok


def W2(b, p):
    return math.ceil(1000 + 1000 * b * 100 / min(p, 60))


def WB(b, p):
    return math.ceil(500 + 100 * b * 100 / min(p, 40))


def prof_from(fns, l2=None, mem=None):
    lat = [[[fn(b, p) for p in GRID] for b in range(1, 33)] for fn in fns]
    return Profile([f"m{i}" for i in range(len(fns))], lat, l2, mem)


def test_worked_examples_identical():
    P = prof_from([W2])
    for r in (300, 700, 2000):
        for mode in ("gpulet", "gpulet+int", "sbp"):
            _check(P, [108_668], [r], 1, mode, (0, 0, 0, 0, 1.0))
    P = prof_from([W2, WB])
    for rates in ([200, 100], [300, 100]):
        _check(P, [108_668, 17_000], rates, 1, "gpulet")


def _inst(rnd, M):
    fns, l2, mem = [], [], []
    for _ in range(M):
        a, c, sat = rnd.randint(200, 5000), rnd.randint(50, 3000), rnd.choice([40, 50, 60, 80, 100])
        fns.append(lambda b, p, a=a, c=c, sat=sat: a + (c * b * 100 + min(p, sat) - 1) // min(p, sat))
        l2.append([[rnd.random() * 0.9 for _ in GRID] for _ in range(6)])
        mem.append([[rnd.random() * 0.9 for _ in GRID] for _ in range(6)])
    P = prof_from(fns, l2, mem)
    return P, [2 * P.L(m, 32, 100) for m in range(M)]


@pytest.mark.parametrize("c", [(0.12, 0.08, 0.21, 0.17, 0.97), (0.068, 0.097, -1.42, 0.71, 1.05)])
@pytest.mark.parametrize("mode", ["gpulet", "gpulet+int", "sbp", "ideal"])
def test_random_instances_identical(mode, c):
    """Second coefficient set: the shape of the B200 fit (c5 > 1, negative c3),
    where the interference-aware batch drops below b_sat."""
    rnd = random.Random(hash(mode) % 1000)
    n = 0
    for _ in range(300 if mode != "ideal" else 40):
        M, N = rnd.randint(1, 6), rnd.randint(1, 4 if mode != "ideal" else 2)
        P, slo = _inst(rnd, M)
        S = sched.Scheduler(P, slo, c, "gpulet")
        rates = [rnd.choice([0, rnd.randint(1, 2 * max(1, S.cap(m, 100)))]) for m in range(M)]
        if not any(rates):
            continue
        _check(P, slo, rates, N, mode, c)
        n += 1
    assert n > 10


def test_fit_interference_matches_oracle():
    import numpy as np
    from oracle import interf
    r = np.random.default_rng(0)
    X = interf.design(r.random(400), r.random(400), r.random(400), r.random(400))
    y = X @ np.array([0.2, 0.1, 0.5, 0.3, 1.0]) + r.normal(0, 0.05, 400)
    np.testing.assert_allclose(gpulet.fit_interference(X, y), interf.fit(X, y), rtol=1e-9, atol=1e-12)
    with pytest.raises(gpulet.GpuletError):
        gpulet.fit_interference(np.tile(X[:1], (50, 1)), np.ones(50))


def test_native_reproduces_worked_sbp_ideal_examples():
    """The hand-derived plans of tests/golden/sched_sbp_ideal_worked.json, through gl_schedule."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "sched_sbp_ideal_worked.json")) as f:
        gold = json.load(f)
    fns = {"W2": W2, "WB": WB}
    for case in gold["cases"]:
        P = prof_from([fns[n] for n in case["profile"]])
        names = ["A", "B"][:len(case["profile"])]
        dump, ok = gpulet.schedule(names, P.lat, None, None, case["slo"], case["rates"], case["gpus"], case["mode"],
                                   (0, 0, 0, 0, 0))
        assert dump == "\n".join(case["dump"]) + "\n", case["name"]
        assert ok == ('"Schedulable"' in case["dump"][-1])
