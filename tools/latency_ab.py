"""Host-observed service latency (submit -> completion visible to gl_poll) of
small batches on a solo gpu-let, median of many (tuning tool for the ring
hand-off / completion path): python tools/latency_ab.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synthgen  # noqa: E402
from tools import common  # noqa: E402


def main():
    import torch
    from paper_2109_01611_b200 import gpulet
    ctx = gpulet.Context(1)
    out = {"lib": os.environ.get("GL_LIB", "in-tree")}
    mids = {m: ctx.load_model(0, m, synthgen.weight_file(m)) for m in ("lenet5", "resnet50", "vgg16", "googlenet")}
    for pct in (20, 40, 80, 100):
        (gid, _n), = ctx.create_gpulets(0, [pct])
        for m, b in (("lenet5", 1), ("resnet50", 1), ("resnet50", 15), ("resnet50", 32), ("vgg16", 8),
                     ("googlenet", 15)):
            x = common.device_input(m, 32)
            y = torch.empty(ctx.model_io(mids[m], 32)[1] // 4, device="cuda")
            out[f"{m}_b{b}_p{pct}_us"] = round(ctx.profile(gid, mids[m], b, x, y, warmup=5, reps=30), 1)
        ctx.destroy_gpulet(gid)
    print(json.dumps(out))
    ctx.close()


if __name__ == "__main__":
    main()
