"""Summarise an `ncu --set full` report into a short text file for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_full_<tag>.txt [--top 25]

Writes the roofline-relevant raw metrics (duration, DRAM bytes, tensor-pipe and
L2/DRAM throughput, occupancy, registers, shared memory), the warp-state stall
breakdown, and the top SASS lines by warp-stall samples (needs -lineinfo for the
CUDA source column).  Runs here (no GPU): `ncu -i` only reads the report.
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "launch__grid_size",
        "launch__block_size", "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, out, top=25):
    lines = []
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units = raw[0], raw[1]
    for i, row in enumerate(raw[2:]):
        lines.append(f"== launch {i}: {row[hdr.index('Kernel Name')]} grid {row[hdr.index('Grid Size')]} "
                     f"block {row[hdr.index('Block Size')]}")
        for k in KEYS:
            if k in hdr:
                j = hdr.index(k)
                lines.append(f"  {k:70s} {row[j]:>16s} {units[j]}")
        for j, k in enumerate(hdr):
            if k.startswith("smsp__average_warp_latency_issue_stalled_") or k.startswith("smsp__average_warps_issue_stalled_"):
                if k.endswith("_per_issue_active.ratio"):
                    try:
                        v = float(row[j])
                    except ValueError:
                        continue
                    if v >= 0.05:
                        lines.append(f"  stall {k:64s} {v:10.3f}")
    for mode in ("sass", "cuda"):
        src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", mode))))
        hi = next((i for i, r in enumerate(src) if "Warp Stall Sampling (All Samples)" in r), None)
        if hi is None:
            continue
        h = src[hi]
        si = h.index("Warp Stall Sampling (All Samples)")
        ai = h.index("Source")
        li = 0
        rows = [r for r in src[hi + 1:] if len(r) > si and r[si].strip().isdigit() and int(r[si]) > 0]
        tot = sum(int(r[si]) for r in rows) or 1
        rows.sort(key=lambda r: -int(r[si]))
        lines.append(f"== top {top} {mode} lines by warp-stall samples (of {tot})")
        for r in rows[:top]:
            lines.append(f"  {100 * int(r[si]) / tot:5.1f}%  {r[li]:>6s}  {r[ai].strip()[:120]}")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    a = sys.argv[1:]
    t = 25
    if "--top" in a:
        i = a.index("--top")
        t = int(a[i + 1])
        del a[i:i + 2]
    main(a[0], a[1], t)
