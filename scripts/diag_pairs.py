"""Diagnose green-context pair residency for one (p, q) pair per process:
    python scripts/diag_pairs.py 50 50
prints the SM ids each executor landed on, or the residency failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthgen  # noqa: E402
from paper_2109_01611_b200 import gpulet  # noqa: E402

p, q = int(sys.argv[1]), int(sys.argv[2])
ctx = gpulet.Context(1)
ctx.load_model(0, "lenet5", synthgen.weight_file("lenet5"))
try:
    got = ctx.create_gpulets(0, [p, q])
    sa, sb = ctx.gpulet_smids(got[0][0]), ctx.gpulet_smids(got[1][0])
    print(p, q, "OK", got, "overlap", sorted(set(sa) & set(sb)), "B", sorted(sb), flush=True)
    for gid, _ in got:
        ctx.destroy_gpulet(gid)
    ctx.close()
except gpulet.GpuletError as e:
    print(p, q, "FAIL", str(e)[:120], flush=True)
    os._exit(1)   # a half-resident executor cannot exit: leave the process
