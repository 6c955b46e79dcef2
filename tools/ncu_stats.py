"""Solo L2 / DRAM utilisation per (model, batch, gpu-let size) from Nsight
Compute, as the paper measures them (§4.4: "L2 utilization
and DRAM bandwidth utilization are the most relevant statistics").

Two phases:
  1. launch (under ncu): one-shot executor launches of every model at the stat
     batches {1,2,4,8,16,32} on n_SM(p) SMs for every gpu-let size p:
       ncu --metrics lts__t_sectors.avg.pct_of_peak_sustained_elapsed,\
dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum \
           -k regex:gl_executor --csv --log-file gpurun_out/ncu_stats.csv \
           python tools/ncu_stats.py launch
  2. apply (anywhere): python tools/ncu_stats.py apply gpurun_out/ncu_stats.csv
     writes l2_util / mem_bw_util (fractions) into profiles/profile_b200.csv.
The launch order is the loop order below, so the CSV rows map back by index.
"""
import csv
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthgen  # noqa: E402
from tools import common  # noqa: E402

L2_METRIC = "lts__t_sectors.avg.pct_of_peak_sustained_elapsed"
DRAM_METRIC = "dram__throughput.avg.pct_of_peak_sustained_elapsed"


def order(sm_counts):
    return [(m, b, gi) for m in common.MODELS for b in common.STAT_B for gi in range(len(common.GRID))]


def launch():
    import torch
    from paper_2109_01611_b200 import gpulet
    nsm = read_sm_counts()
    ctx = gpulet.Context(1)
    mids = {m: ctx.load_model(0, m, synthgen.weight_file(m)) for m in common.MODELS}
    xs = {m: common.device_input(m, 32) for m in common.MODELS}
    ys = {m: torch.empty(ctx.model_io(mids[m], 32)[1] // 4, device="cuda") for m in common.MODELS}
    torch.cuda.synchronize()
    for m, b, gi in order(nsm):
        ctx.run_once(mids[m], b, xs[m], ys[m], nsm[gi], False)
    ctx.close()


def read_sm_counts():
    with open(common.PROFILE_CSV) as f:
        rows = list(csv.DictReader(f))
    out = {}
    for r in rows:
        out[common.GRID.index(int(r["partition_pct"]))] = int(r["sm_count"])
    return [out[g] for g in range(len(common.GRID))]


def apply(path):
    with open(path) as f:
        text = f.read()
    lines = [ln for ln in text.splitlines() if ln.startswith('"')]
    rdr = csv.DictReader(io.StringIO("\n".join(lines)))
    vals = {}
    for r in rdr:
        if "gl_executor" not in r.get("Kernel Name", ""):
            continue
        k = int(r["ID"])
        vals.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ids = sorted(vals)
    seq = order(None)
    if len(ids) != len(seq):
        raise SystemExit(f"{len(ids)} profiled launches, expected {len(seq)}")
    stat = {}
    for k, (m, b, gi) in zip(ids, seq):
        stat[(m, b, common.GRID[gi])] = (vals[k].get(L2_METRIC, 0.0) / 100.0, vals[k].get(DRAM_METRIC, 0.0) / 100.0)
    with open(common.PROFILE_CSV) as f:
        rows = list(csv.DictReader(f))
    for r in rows:
        key = (r["model"], int(r["batch"]), int(r["partition_pct"]))
        if key in stat:
            r["l2_util"] = f"{min(1.0, stat[key][0]):.6f}"
            r["mem_bw_util"] = f"{min(1.0, stat[key][1]):.6f}"
    with open(common.PROFILE_CSV, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    print(f"applied {len(stat)} ncu rows to {common.PROFILE_CSV}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "apply":
        apply(sys.argv[2])
    else:
        launch()
