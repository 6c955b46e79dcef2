"""Harness helpers shared by bench.py and tools/*.py (not part of libgpulet).

Device inputs are built from synthgen (seeded) and moved to the GPU once; all
compute goes through libgpulet's C-ABI via the thin binding.
"""
import csv
import json
import os

import numpy as np

import synthgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRID = (20, 40, 50, 60, 80, 100)
STAT_B = (1, 2, 4, 8, 16, 32)
MODELS = synthgen.MODELS
PROFILE_CSV = os.path.join(ROOT, "profiles", "profile_b200.csv")
COEFFS_JSON = os.path.join(ROOT, "profiles", "coeffs_b200.json")


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


def load_profile(path=PROFILE_CSV, slo_mode="rule"):
    """The profile as libgpulet parses and envelopes it (gl_profile_load, C4.1) and the
    SLOs it derives (gl_workload_rates, C4.2): dict lat [m][b-1][gi] (µs), l2, mem
    [m][si][gi], sm {p: SMs}, slo [m] (µs).  No scheduling arithmetic in Python."""
    from paper_2109_01611_b200 import gpulet
    lat, l2, mem, sm = gpulet.profile_load(path)
    slo = gpulet.workload_rates(lat, "equal", 1.0, 1, slo_mode)[0]
    return {"lat": lat.tolist(), "l2": l2.tolist(), "mem": mem.tolist(), "sm": dict(zip(GRID, sm.tolist())),
            "slo": slo, "lat_np": lat}


def scenario_rates(prof, scen, x=1.0, n_gpus=1, slo_mode="rule"):
    """Scenario rates at multiplier x (gl_workload_rates: C4.3-C4.4, scaled natively)."""
    from paper_2109_01611_b200 import gpulet
    return gpulet.workload_rates(prof["lat_np"], scen, x, n_gpus, slo_mode)[1]


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
