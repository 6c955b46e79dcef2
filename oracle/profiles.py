"""C4 profile post-processing, SLO rule, rate scaling, scenarios (ORACLE).

* min-envelope (C4.1): L*(b,p) = min over b' >= b, p' <= p of L_raw(b',p') —
  realisable (pad the batch / run on fewer SMs); enforces the monotonicity of
  S:41-42.
* SLO rule (C4.2): SLO_m = 2 * L*_m(32, 100 %) — "set by doubling the solo
  execution latency" at batch 32.
* rate scaling (C4.3): paper rates * SLO_paper / SLO_B200 (BERT uses ResNet's).
* scenarios (C4.4): Table `tab:particular-scenarios`, game,
  traffic, mix6.
Pinned in tests/test_oracle_sched.py (idempotence, monotonicity, SLO rule =>
b_sat(100) = 32).
"""
import csv
import io

GRID = (20, 40, 50, 60, 80, 100)
BMAX = 32
NAMES = ("lenet5", "googlenet", "resnet50", "ssd_mobilenet_v1", "vgg16", "bert_base")
SHORT = ("le", "goo", "res", "ssd", "vgg", "bert")
PAPER_SLO_MS = {"googlenet": 44, "lenet5": 5, "resnet50": 95, "ssd_mobilenet_v1": 136,
                "vgg16": 130}                                   # Table tab:ml-models


def envelope(lat):
    """lat[b-1][gi] -> min-envelope over (b' >= b, p' <= p)."""
    out = [[0] * len(GRID) for _ in range(BMAX)]
    for b in range(BMAX):
        for g in range(len(GRID)):
            out[b][g] = min(lat[bb][gg] for bb in range(b, BMAX) for gg in range(0, g + 1))
    return out


def slo_rule(lat_env):
    return 2 * lat_env[BMAX - 1][GRID.index(100)]


def scale_rates(paper_rates, slo_b200_us):
    """rates[m] * SLO_paper / SLO_B200, int floor; BERT reuses ResNet's scale."""
    out = []
    for name, r in zip(NAMES, paper_rates):
        ref = name if name in PAPER_SLO_MS else "resnet50"
        num = r * PAPER_SLO_MS[ref] * 1000
        out.append(num // slo_b200_us[NAMES.index(ref)])
    return out


SCENARIOS = {
    "equal": (50, 50, 50, 50, 50, 50),
    "long-only": (0, 0, 100, 100, 100, 100),
    "short-skew": (100, 100, 100, 50, 50, 50),
    "mix6": (50, 50, 50, 50, 50, 50),
}


def app_rates(app, r):
    """Model-level rates of an application at app rate r."""
    if app == "game":
        return (6 * r, 0, r, 0, 0, 0)
    if app == "traffic":
        return (0, r, 0, r, r, 0)
    raise ValueError(app)


def read_profile_csv(text):
    """CSV `model,batch,partition_pct,sm_count,latency_us,l2_util,mem_bw_util`
    -> (lat[m][b-1][gi] int, l2[m][si][gi], mem[m][si][gi]) (blank stats allowed)."""
    M = len(NAMES)
    lat = [[[None] * 6 for _ in range(BMAX)] for _ in range(M)]
    stat_b = (1, 2, 4, 8, 16, 32)
    l2 = [[[0.0] * 6 for _ in stat_b] for _ in range(M)]
    mem = [[[0.0] * 6 for _ in stat_b] for _ in range(M)]
    for i, row in enumerate(csv.DictReader(io.StringIO(text))):
        m = NAMES.index(row["model"])
        b, p = int(row["batch"]), int(row["partition_pct"])
        lat[m][b - 1][GRID.index(p)] = int(row["latency_us"])
        if row.get("l2_util") not in (None, "") and b in stat_b:
            l2[m][stat_b.index(b)][GRID.index(p)] = float(row["l2_util"])
            mem[m][stat_b.index(b)][GRID.index(p)] = float(row["mem_bw_util"])
    return lat, l2, mem
