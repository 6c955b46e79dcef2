"""Compare per-step device times of two oneshot traces: python tools/cmp_trace.py a.json b.json"""
import json
import sys

a, b = (json.load(open(p)) for p in sys.argv[1:3])
print(f"{a['model']} b={a['batch']}: {a['total_us']} -> {b['total_us']} us")
for x, y in zip(a["rows"], b["rows"]):
    d = y["us"] - x["us"]
    if abs(d) > 1.0:
        print(f"  step {x['step']:3d} {x['op']:>12} {x['gflop']:7.3f} GF  {x['us']:8.2f} -> {y['us']:8.2f}  ({d:+.2f})")
