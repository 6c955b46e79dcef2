"""C4 inputs of the scheduler from SPEC-format files (ORACLE — test infrastructure only).

What the native `gl_profile_load` / `gl_workload_rates` / `gl_schedule_files`
(include/gpulet.h) must compute, restated plainly from the paper and SURVEY
§8(c) C4 (readings in DESIGN.md §2):

* profile CSV (SPEC S:130 + sm_count): one row per (model, batch 1..32,
  p in {20,40,50,60,80,100}); latency in µs (`latency_us`) or ms
  (`latency_ms`, SPEC's unit), converted exactly (fractions.Fraction) and
  rounded up to whole µs (C2.1);
* C4.1 min-envelope L*(b,p) = min over b' >= b, p' <= p of L(b',p') — or, in
  strict mode, SPEC S:41-42's monotonicity check (a violation is a data error);
* C4.2 SLOs: rule SLO_m = 2 L*_m(32, 100 %), or Table
  tab:ml-models constants (BERT-base, absent from the paper, 95 ms);
* C4.3/C4.4 rates: the paper's scenario rates (Table tab:particular-scenarios
  P:800-806, game P:787, traffic P:788-790) times SLO_paper/SLO_B200 of a
  reference model (the model itself; ResNet-50 for BERT; the app-SLO model for
  an application, DESIGN R23) times x, floored, times num_gpus.  The product is
  evaluated in IEEE double as ((base * paper_us) * x) / slo_us — the order the
  C-ABI documents — so both sides floor the same double;
* the plan: oracle.sched on those tables, preceded by a header line.

Pins (tests/test_oracle_workload.py): the paper's Table constants; game's
6:1 and traffic's 1:1:1 compositions at every x; rates equal to the scenario
rates where the profile's SLO equals the paper's (scale 1); a hand-computed
rule-mode example; exact decimal conversion (0.1 ms -> 100 µs, not 101);
the envelope's closed-form properties; error kinds on malformed files.
"""
import json
import math
from fractions import Fraction

from oracle import sched as osched

NAMES = ("lenet5", "googlenet", "resnet50", "ssd_mobilenet_v1", "vgg16", "bert_base")
GRID = (20, 40, 50, 60, 80, 100)
STAT_B = (1, 2, 4, 8, 16, 32)
BMAX = 32
SM_DEFAULT = (30, 60, 74, 88, 118, 148)    # exact shares of 148 SMs, in SM pairs (DESIGN R15)
PAPER_SLO_MS = (5, 44, 95, 136, 130, 95)    # P:750-756 (le, goo, res, ssd, vgg) + BERT 95 ms
SCENARIOS = {
    "equal": ((50, 50, 50, 50, 50, 50), None),
    "mix6": ((50, 50, 50, 50, 50, 50), None),
    "long-only": ((0, 0, 100, 100, 100, 100), None),
    "short-skew": ((100, 100, 100, 50, 50, 50), None),
    "game": ((600, 0, 100, 0, 0, 0), 2),        # app rate 100: 6 LeNet + 1 ResNet-50 each
    "traffic": ((0, 100, 0, 100, 100, 0), 3),   # SSD -> GoogLeNet + VGG-16; app SLO = SSD's
}


class WorkloadError(Exception):
    """kind in {"parse", "data", "arg"} (GL_E_PARSE / GL_E_DATA / GL_E_ARG)."""

    def __init__(self, kind, msg):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


def _ceil_decimal(text, scale):
    try:
        v = Fraction(text.strip().lstrip("+")) * scale
    except (ValueError, ZeroDivisionError):
        return None
    if v < 0:
        return None
    return math.ceil(v)


def parse_profile(text, strict=False):
    """-> dict(lat=[m][b-1][gi] int µs (enveloped unless strict), l2/mem=[m][si][gi], sm=[6])."""
    lines = text.splitlines()
    rows = [(i + 1, ln) for i, ln in enumerate(lines) if ln.strip()]
    if not rows:
        raise WorkloadError("parse", "empty profile")
    head = [h.strip() for h in rows[0][1].split(",")]
    col = {h: k for k, h in enumerate(head)}
    if not {"model", "batch", "partition_pct"} <= set(col) or not ({"latency_us", "latency_ms"} & set(col)):
        raise WorkloadError("parse", "header")
    lat = [[[None] * 6 for _ in range(BMAX)] for _ in NAMES]
    l2 = [[[0.0] * 6 for _ in STAT_B] for _ in NAMES]
    mem = [[[0.0] * 6 for _ in STAT_B] for _ in NAMES]
    sm = [None] * 6
    for lineno, ln in rows[1:]:
        f = [x.strip() for x in ln.split(",")]
        if len(f) != len(head):
            raise WorkloadError("parse", f"line {lineno}: field count")
        if f[col["model"]] not in NAMES:
            raise WorkloadError("data", f"line {lineno}: unknown model")
        m = NAMES.index(f[col["model"]])
        try:
            b, p = int(f[col["batch"]]), int(f[col["partition_pct"]])
        except ValueError:
            raise WorkloadError("parse", f"line {lineno}: batch/partition")
        if not 1 <= b <= BMAX:
            raise WorkloadError("data", f"line {lineno}: batch")
        if p not in GRID:
            raise WorkloadError("data", f"line {lineno}: partition off grid")
        g = GRID.index(p)
        us = (_ceil_decimal(f[col["latency_us"]], 1) if "latency_us" in col
              else _ceil_decimal(f[col["latency_ms"]], 1000))
        if us is None:
            raise WorkloadError("parse", f"line {lineno}: latency")
        if us <= 0:
            raise WorkloadError("data", f"line {lineno}: latency must be positive")
        if lat[m][b - 1][g] is not None:
            raise WorkloadError("data", f"line {lineno}: duplicate row")
        lat[m][b - 1][g] = us
        if "sm_count" in col and f[col["sm_count"]] != "":
            n = int(f[col["sm_count"]])
            if n < 1 or (sm[g] is not None and sm[g] != n):
                raise WorkloadError("data", f"line {lineno}: sm_count")
            sm[g] = n
        if b in STAT_B:
            si = STAT_B.index(b)
            for key, dst in (("l2_util", l2), ("mem_bw_util", mem)):
                if key in col and f[col[key]] != "":
                    v = float(f[col[key]])
                    if not 0.0 <= v <= 1.0:
                        raise WorkloadError("data", f"line {lineno}: utilisation")
                    dst[m][si][g] = v
    for m in range(len(NAMES)):
        for b in range(BMAX):
            for g in range(6):
                if lat[m][b][g] is None:
                    raise WorkloadError("data", f"missing row {NAMES[m]},{b + 1},{GRID[g]}")
    sm = [sm[g] if sm[g] is not None else SM_DEFAULT[g] for g in range(6)]
    if strict:
        for m in range(len(NAMES)):
            for b in range(BMAX):
                for g in range(6):
                    if (b > 0 and lat[m][b][g] < lat[m][b - 1][g]) or (g > 0 and lat[m][b][g] > lat[m][b][g - 1]):
                        raise WorkloadError("data", f"monotonicity at {NAMES[m]},{b + 1},{GRID[g]}")
    else:
        lat = [envelope(lat[m]) for m in range(len(NAMES))]
    return {"lat": lat, "l2": l2, "mem": mem, "sm": sm}


def envelope(lat):
    """C4.1, written as its definition: min over b' >= b and p' <= p."""
    return [[min(lat[bb][gg] for bb in range(b, BMAX) for gg in range(g + 1)) for g in range(6)]
            for b in range(BMAX)]


def slos(lat_env, slo_mode):
    if slo_mode == "rule":
        return [2 * lat_env[m][BMAX - 1][GRID.index(100)] for m in range(len(NAMES))]
    if slo_mode == "table":
        return [ms * 1000 for ms in PAPER_SLO_MS]
    raise WorkloadError("arg", "slo_mode")


PAPER_APP_SLO_MS = {"game": 95, "traffic": 136}


def traffic_stage_slos(lat_env, slo_mode="rule", handoff_us=0):
    """F3 `traffic` as a two-stage chain (DESIGN R28).  The application SLO is "the
    longest model inference latency" of the app doubled: 2 max over
    {SSD, GoogLeNet, VGG-16} of L*(32, 100 %) in rule mode, 136 ms in table mode.
    The detector stage gets the share of it that its solo latency has of the two
    stages' (the slower recogniser counts: they run in parallel):
    s1 = floor(s_app L_ssd / (L_ssd + max(L_goo, L_vgg))), all at (32, 100 %).
    Returns (s_app, s1); the recognisers' budget from their spawn is
    s_app - s1 - handoff_us."""
    g = GRID.index(100)
    L = {m: lat_env[NAMES.index(m)][BMAX - 1][g] for m in ("ssd_mobilenet_v1", "googlenet", "vgg16")}
    if slo_mode == "rule":
        s_app = 2 * max(L.values())
    elif slo_mode == "table":
        s_app = PAPER_APP_SLO_MS["traffic"] * 1000
    else:
        raise WorkloadError("arg", "slo_mode")
    l2 = max(L["googlenet"], L["vgg16"])
    s1 = (s_app * L["ssd_mobilenet_v1"]) // (L["ssd_mobilenet_v1"] + l2)
    if s_app - s1 - handoff_us <= 0:
        raise WorkloadError("arg", "handoff_us")
    return s_app, s1


def chain_workload(lat_env, slo_mode, x=1.0, num_gpus=1, handoff_us=0):
    """Scenario "traffic-chain": per-model SLOs of the plan (SSD s1; GoogLeNet and VGG-16
    s_app - s1 - handoff_us, their budget from the spawn) and rates: traffic's 100 req/s
    per model scaled by the application's SLO, floor((100 * 136 ms * x) /
    s_app) * num_gpus (C4.3 with the app SLO as the reference, R23/R28)."""
    if not (x >= 0.0 and math.isfinite(x)):
        raise WorkloadError("arg", "x")
    s_app, s1 = traffic_stage_slos(lat_env, slo_mode, handoff_us)
    slo = slos(lat_env, slo_mode)
    rates = [0] * len(NAMES)
    for m in ("ssd_mobilenet_v1", "googlenet", "vgg16"):
        i = NAMES.index(m)
        slo[i] = s1 if m == "ssd_mobilenet_v1" else s_app - s1 - handoff_us
        rates[i] = math.floor(float(100 * PAPER_APP_SLO_MS["traffic"] * 1000) * x / float(s_app)) * num_gpus
    return slo, rates, s_app


def scenario_rates(scenario, slo_us, x=1.0, num_gpus=1):
    """Returns (rates, base).  rate_m = floor(((base_m * paper_us_ref) * x) / slo_us_ref) * num_gpus."""
    if scenario not in SCENARIOS:
        raise WorkloadError("arg", "scenario")
    if not (x >= 0.0 and math.isfinite(x)):
        raise WorkloadError("arg", "x")
    base, app = SCENARIOS[scenario]
    return scale_base(base, app, slo_us, x, num_gpus), list(base)


def scale_base(base, app, slo_us, x=1.0, num_gpus=1):
    """C4.3 for any paper-scale rate vector (app = index of the app-SLO model, or None)."""
    if not (x >= 0.0 and math.isfinite(x)):
        raise WorkloadError("arg", "x")
    out = []
    for m in range(len(NAMES)):
        ref = app if app is not None else (2 if NAMES[m] == "bert_base" else m)
        v = float(base[m] * PAPER_SLO_MS[ref] * 1000) * x / float(slo_us[ref])
        out.append(math.floor(v) * num_gpus)
    return out


def schedule_files(profile_text, coeffs_text, workload_text):
    """-> (output text, schedulable) as gl_schedule_files writes it."""
    try:
        W = json.loads(workload_text)
    except ValueError as e:
        raise WorkloadError("parse", str(e))
    strict = W.get("envelope", True) is False
    prof = parse_profile(profile_text, strict=strict)
    N = W.get("num_gpus", 1)
    mode = W.get("mode", "gpulet")
    if mode not in ("gpulet", "gpulet+int", "sbp", "ideal", "sbp50"):
        raise WorkloadError("arg", "mode")
    slo_mode = W.get("slo_mode", "rule")
    slo = slos(prof["lat"], slo_mode)
    given = [k for k in ("scenario", "base_rates", "rates", "models") if k in W]
    if len(given) != 1:
        raise WorkloadError("arg", "exactly one of scenario, base_rates, rates, models")
    truncated = None
    app_slo = None
    if W.get("scenario") == "traffic-chain":
        slo, rates, app_slo = chain_workload(prof["lat"], slo_mode, float(W.get("x", 1.0)), N,
                                             int(W.get("handoff_us", 0)))
        base = [0, 100, 0, 100, 100, 0]
        truncated = next((m for m in range(len(NAMES)) if base[m] > 0 and rates[m] == 0), None)
    elif "scenario" in W or "base_rates" in W:
        if "scenario" in W:
            rates, base = scenario_rates(W["scenario"], slo, float(W.get("x", 1.0)), N)
        else:
            base = [int(v) for v in W["base_rates"]]
            rates = scale_base(base, None, slo, float(W.get("x", 1.0)), N)
        truncated = next((m for m in range(len(NAMES)) if base[m] > 0 and rates[m] == 0), None)
    elif "rates" in W:
        rates = [int(r) for r in W["rates"]]
    else:
        rates = [0] * len(NAMES)
        for e in W["models"]:
            m = NAMES.index(e["name"])
            rates[m] = int(e["rate"])
            if "slo_ms" in e:
                slo[m] = _ceil_decimal(str(e["slo_ms"]), 1000)
    coeffs = None
    if coeffs_text is not None:
        coeffs = tuple(float(c) for c in json.loads(coeffs_text)["coeffs"])
    hd = {"slo_us": slo, "rates": rates, "num_gpus": N, "mode": mode, "slo_mode": slo_mode}
    if app_slo is not None:
        hd["app_slo_us"] = app_slo
    head = json.dumps(hd, separators=(",", ":")) + "\n"
    if truncated is not None:
        return head + json.dumps({"verdict": "NotSchedulable", "failed_model": NAMES[truncated],
                                  "reason": "rate_truncated"}, separators=(",", ":")) + "\n", False
    P = osched.Profile(NAMES, prof["lat"], prof["l2"], prof["mem"], sm=prof["sm"])
    if mode == "ideal":
        plan = osched.ideal(P, slo, rates, N, "gpulet+int", coeffs if coeffs is not None else (0.0,) * 5)
    else:
        plan = osched.schedule(P, slo, rates, N, mode, coeffs)
    return head + plan.dump, plan.ok
