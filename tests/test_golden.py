"""Golden fixtures (tests/golden/*.json, each carrying its citation) checked
against the oracle.  Values are the paper's (PAPER.md tables/text), SPEC.md's
worked examples, or SURVEY.md's hand-derived examples -- never produced by the
CUDA path or by the oracle itself."""
import json
import math
import os
from itertools import combinations_with_replacement, product

import pytest

from oracle import profiles, sched
from oracle.sched import GRID, Profile, Scheduler

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        d = json.load(f)
    assert d.get("cite"), f"{name} has no citation"
    return d


def test_every_fixture_cites_its_source():
    for fn in sorted(os.listdir(GOLDEN)):
        if fn.endswith(".json"):
            assert "P:" in load(fn)["cite"] or "S:" in load(fn)["cite"] or "SURVEY" in load(fn)["cite"]


def test_paper_slo_table_is_twice_the_batch32_latency():
    """the table's SLOs are 2 x L(32) -- the oracle's SLO rule gives back
    the table from profiles whose L(32,100) is half of it, at any curve shape."""
    d = load("paper_tab_ml_models.json")
    for m, slo_ms in d["slo_ms"].items():
        half = slo_ms * 1000 // d["rule_factor"]
        for shape in (lambda b, p: b * 100 / p, lambda b, p: 1 + b * 10 / p, lambda b, p: math.sqrt(b) * 100 / p):
            raw = [[max(1, round(half * shape(b, p) / shape(32, 100))) for p in GRID] for b in range(1, 33)]
            env = profiles.envelope(raw)
            assert env[31][5] == half
            assert profiles.slo_rule(env) == slo_ms * 1000, m


def test_paper_apps_composition():
    d = load("paper_apps.json")
    names = ["lenet5", "googlenet", "resnet50", "ssd_mobilenet_v1", "vgg16", "bert_base"]
    for app in ("game", "traffic"):
        want = tuple(d[app].get(n, 0) * 7 for n in names)
        assert profiles.app_rates(app, 7) == want
    # the app SLO is the SLO of its longest model (Table tab:ml-models)
    slo = load("paper_tab_ml_models.json")["slo_ms"]
    for app in ("game", "traffic"):
        models = [n for n in names if d[app].get(n)]
        assert d[app]["slo_ms"] == max(slo[n] for n in models) == slo[d[app]["slo_model"]]


def test_paper_ideal_case_count():
    d = load("paper_ideal_cases.json")
    lay = [tuple(x) for x in d["layouts"]]
    assert tuple(sched.LAYOUTS) == tuple(lay)
    assert len(list(product(range(len(lay)), repeat=d["gpus"]))) == d["ordered_cases"]       # 4^4
    assert len(list(combinations_with_replacement(range(len(lay)), d["gpus"]))) == d["multiset_cases"]
    for l in lay:
        assert sum(l) <= 100 and all(p in GRID for p in l)


def _prof(fns):
    lat = [[[fn(b, p) for p in GRID] for b in range(1, 33)] for fn in fns]
    return Profile([f"m{i}" for i in range(len(fns))], lat, None, None)


def test_spec_bsat_S80():
    d = load("spec_bsat_S80.json")
    P = _prof([lambda b, p: d["latency_us_per_batch"] * b])
    for c in d["cases"]:
        assert Scheduler(P, [c["slo_us"]], None, "gpulet").b_sat(0, c["p"]) == c["b_sat"]


def test_survey_knee_W1():
    d = load("survey_knee_W1.json")
    for c in d["curves"]:
        assert sched.knee(c["rates"]) == c["knee"]
        k = sched.curvatures(c["rates"])
        for key, nd in (("curv4", 4), ("curv3", 3)):
            for p, v in c.get(key, {}).items():
                assert round(k[int(p)], nd) == v


def test_spec_factor_S170():
    d = load("spec_factor_S170.json")
    l2 = [[[d["victim"]["l2"]] * 6 for _ in range(6)]]
    mem = [[[d["victim"]["mem"]] * 6 for _ in range(6)]]
    P = Profile(["x"], [[[d["solo_us"]] * 6 for _ in range(32)]], l2, mem)
    part = (d["partner"]["l2"], d["partner"]["mem"])
    S = Scheduler(P, [10**9], tuple(d["coeffs"]), "gpulet+int")
    f = S.factor(0, 4, 50, part)
    assert f == d["factor_permille"]
    assert S.leff(0, 4, 50, f) == d["leff_us"]
    S0 = Scheduler(P, [10**9], tuple(d["clamp_case"]["coeffs"]), "gpulet+int")
    assert S0.factor(0, 4, 50, part) == d["clamp_case"]["factor_permille"]


def test_survey_W2_plans():
    d = load("survey_W2_plans.json")
    W2 = lambda b, p: math.ceil(1000 + 1000 * b * 100 / min(p, 60))   # noqa: E731
    P = _prof([W2])
    slo = [2 * W2(32, 100)]
    assert slo == [d["slo_us"]]
    S = Scheduler(P, slo, None, "gpulet")
    assert [S.b_sat(0, p) for p in GRID] == d["b_sat"]
    assert S.curve(0) == d["curve"]
    assert round(sched.curvatures(S.curve(0))[60], 4) == d["curv60"]
    assert S.p_eff(0) == d["p_eff"]
    for r, p in d["p_req"].items():
        assert S.p_req(0, int(r)) == p
    for c in d["plans"]:
        plan = sched.schedule(P, slo, [c["rate"]], c["gpus"], "gpulet")
        assert plan.ok == c["ok"]
        if not c["ok"] or c["gpus"] != 1:
            continue
        gl = [json.loads(l) for l in plan.dump.splitlines()[:-1]]
        for k, g in (("slot0", gl[0]), ("slot1", gl[1])):
            if k in c:
                ln = g["lanes"][0]
                assert (g["size"], ln["rate"], ln["batch"], ln["exec_us"]) == \
                    (c[k]["size"], c[k]["rate"], c[k]["batch"], c[k]["exec_us"])


def test_top1_golden_files_match_oracle():
    """tests/golden/top1_*.npz (scripts/make_top1_golden.py) exist for every model and
    their first LeNet-5 batch equals a fresh oracle forward (the files are oracle output)."""
    import numpy as np
    import synthgen
    from oracle import models as om
    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    for m in synthgen.MODELS:
        g = np.load(os.path.join(gdir, f"top1_{m}.npz"))
        n = 1024 if m == "lenet5" else 256
        assert len(g["batch_ids"]) * int(g["batch"]) == n
    g = np.load(os.path.join(gdir, "top1_lenet5.npz"))
    b = int(g["batch"])
    ref = om.forward("lenet5", synthgen.weights("lenet5"), synthgen.model_input("lenet5", b, int(g["batch_ids"][0])))
    assert np.array_equal(g["logits"][:b], ref["logits"].astype(np.float32))
