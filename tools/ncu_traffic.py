"""DRAM traffic per executor launch from an ncu metrics CSV (roofline `traffic`).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:gl_executor --csv --log-file gpurun_out/ncu_traffic_<m>_b<b>.csv \
        python tools/oneshot.py --model <m> --batch <b> --reps 3
    python tools/ncu_traffic.py gpurun_out/ncu_traffic_<m>_b<b>.csv <m> <b>
writes profiles/ncu_<m>_b<b>.json {dram_bytes, dram_read, dram_write, ncu_us} (median
over the profiled launches; ncu timings are serialised, cold-cache: shares only).
"""
import csv
import io
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, model, batch):
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith('"')]
    per = {}
    for r in csv.DictReader(io.StringIO("\n".join(lines))):
        if "gl_executor" not in r.get("Kernel Name", ""):
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
                 "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1)
        per.setdefault(int(r["ID"]), {})[r["Metric Name"]] = v * scale
    rd = [d.get("dram__bytes_read.sum", 0) for d in per.values()]
    wr = [d.get("dram__bytes_write.sum", 0) for d in per.values()]
    us = [d.get("gpu__time_duration.sum", 0) for d in per.values()]
    out = {"model": model, "batch": int(batch), "launches": len(per), "dram_read": statistics.median(rd),
           "dram_write": statistics.median(wr), "dram_bytes": statistics.median([a + b for a, b in zip(rd, wr)]),
           "ncu_us": statistics.median(us), "source": os.path.basename(path)}
    dst = os.path.join(ROOT, "profiles", f"ncu_{model}_b{batch}.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(*sys.argv[1:4])
