"""Harness helpers shared by bench.py and tools/*.py (not part of libgpulet).

Device inputs are built from synthgen (seeded) and moved to the GPU once; all
compute goes through libgpulet's C-ABI via the thin binding.
"""
import csv
import io
import json
import os

import numpy as np

import synthgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRID = (20, 40, 50, 60, 80, 100)
SM_OF = {20: 32, 40: 56, 50: 72, 60: 92, 80: 116, 100: 148}
STAT_B = (1, 2, 4, 8, 16, 32)
MODELS = synthgen.MODELS
PROFILE_CSV = os.path.join(ROOT, "profiles", "profile_b200.csv")
COEFFS_JSON = os.path.join(ROOT, "profiles", "coeffs_b200.json")
PAPER_SLO_MS = {"googlenet": 44, "lenet5": 5, "resnet50": 95, "ssd_mobilenet_v1": 136, "vgg16": 130}


def device_input(model, batch, batch_id=0):
    """Resident device input in the ABI layout (C padded 3 -> 8 for images)."""
    import torch
    x = synthgen.model_input(model, batch, batch_id)
    if model == "bert_base":
        return torch.from_numpy(x).cuda()
    if model != "lenet5":
        x = synthgen.pad_channels(x, 8)
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()


def host_input(model, batch, batch_id=0):
    """Pinned host copy of the same input (e2e leg)."""
    import torch
    x = synthgen.model_input(model, batch, batch_id)
    if model != "bert_base" and model != "lenet5":
        x = synthgen.pad_channels(x, 8)
    if model == "bert_base":
        t = torch.from_numpy(np.ascontiguousarray(x))
    else:
        t = torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16)
    return t.pin_memory()


def write_profile_csv(path, lat, nsm, l2, mem):
    """lat[m][b-1][gi] int us; l2/mem[m][si][gi]; CSV (SPEC S:130 + sm_count)."""
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["model", "batch", "partition_pct", "sm_count", "latency_us", "l2_util", "mem_bw_util"])
        for m, name in enumerate(MODELS):
            for b in range(1, 33):
                for gi, p in enumerate(GRID):
                    if b in STAT_B:
                        si = STAT_B.index(b)
                        w.writerow([name, b, p, nsm[gi], lat[m][b - 1][gi], f"{l2[m][si][gi]:.6f}",
                                    f"{mem[m][si][gi]:.6f}"])
                    else:
                        w.writerow([name, b, p, nsm[gi], lat[m][b - 1][gi], "", ""])


def read_profile_csv(path):
    from oracle import profiles  # CSV parsing only; no scheduling arithmetic
    with open(path) as f:
        return profiles.read_profile_csv(f.read())


def envelope(lat):
    """C4.1 min-envelope, applied by the harness before scheduling (as the
    oracle does); realisable by padding the batch or using fewer SMs."""
    out = [[0] * 6 for _ in range(32)]
    for b in range(31, -1, -1):
        for g in range(6):
            v = lat[b][g]
            if b + 1 < 32:
                v = min(v, out[b + 1][g])
            if g > 0:
                v = min(v, out[b][g - 1])
            out[b][g] = v
    return out


def slos_from(lat_env):
    """SLO_m = 2 L*(32, 100 %)."""
    return [2 * lat_env[m][31][5] for m in range(len(lat_env))]


def scenario_rates(name, slo_us, x=1.0):
    """Rates of a scenario, scaled by SLO_paper/SLO_B200 (C4.3) and multiplier x."""
    base = {"equal": (50,) * 6, "mix6": (50,) * 6, "long-only": (0, 0, 100, 100, 100, 100),
            "short-skew": (100, 100, 100, 50, 50, 50)}
    app_ref = None
    if name.startswith("game"):
        r = (6, 0, 1, 0, 0, 0)
        base_r = [v * 100 for v in r]
        app_ref = "resnet50"           # app SLO = ResNet-50's
    elif name.startswith("traffic"):
        base_r = [0, 100, 0, 100, 100, 0]
        app_ref = "ssd_mobilenet_v1"   # app SLO = SSD's 136 ms
    else:
        base_r = list(base[name])
    if app_ref is not None:
        # an application keeps its composition (6 LeNet + 1 ResNet per
        # game request): one B200 scale for all its models, the app-SLO model's
        s = PAPER_SLO_MS[app_ref] * 1000.0 / slo_us[MODELS.index(app_ref)]
        return [int(r * s * x) for r in base_r]
    out = []
    for m, r in enumerate(base_r):
        ref = MODELS[m] if MODELS[m] in PAPER_SLO_MS else "resnet50"
        s = PAPER_SLO_MS[ref] * 1000.0 / slo_us[MODELS.index(ref)]
        out.append(int(r * s * x))
    return out


def load_coeffs(path=COEFFS_JSON):
    if os.path.exists(path):
        with open(path) as f:
            return tuple(json.load(f)["coeffs"])
    return (0.0, 0.0, 0.0, 0.0, 1.0)


def parse_plan(dump):
    gls, verdict = [], None
    for line in dump.splitlines():
        d = json.loads(line)
        if "verdict" in d:
            verdict = d
        else:
            gls.append(d)
    return gls, verdict
