"""gl_serve on live gpu-lets: every request completes,
and in end-to-end mode the outputs that land in the pinned host ring -- by the
zero-copy path (LeNet: the executor reads/writes the host ring itself) and by
the async copy path (ResNet-50: H2D / D2H on the lane's stream) -- match the
CPU oracle."""
import numpy as np
import pytest

import synthgen
from oracle import models as omodels
from tests.gpu_util import REL_TOL, rel_err

pytestmark = pytest.mark.gpu


def test_serve_e2e_zero_copy_and_copy_paths():
    import torch
    from paper_2109_01611_b200 import gpulet
    from tools import common
    ctx = gpulet.Context(1)
    try:
        mids = {m: ctx.load_model(0, m, synthgen.weight_file(m)) for m in ("lenet5", "resnet50")}
        (g0, _n0), (g1, _n1) = ctx.create_gpulets(0, [20, 80])
        lanes, refs = [], {}
        slots = {"lenet5": 32, "resnet50": 4}
        for gid, m, slot, b in ((g0, "lenet5", 0, 8), (g1, "resnet50", 1, 2)):
            inb, outb = ctx.model_io(mids[m], 32)
            ib, ob = inb // 32, outb // 32
            xh = common.host_input(m, slots[m])                      # pinned, one request per slot
            yh = torch.zeros(slots[m] * ob // 4, dtype=torch.float32).pin_memory()
            x = common.device_input(m, 32)
            y = torch.empty(outb // 4, device="cuda")
            lanes.append(dict(gpulet=gid, model_id=mids[m], model_slot=slot, batch=b, duty_us=200, weight=1,
                              drop_us=0, x=x, y=y, x_host=xh, y_host=yh, in_req_bytes=ib, out_req_bytes=ob,
                              host_slots=slots[m], x2=common.device_input(m, 32),
                              y2=torch.empty(outb // 4, device="cuda")))
            refs[m] = (yh, ob // 4)
        # 64 LeNet requests (model slot 0) and 6 ResNet requests (slot 1), arrivals in us
        t = np.concatenate([np.arange(64) * 30, 100 + np.arange(6) * 3000]).astype(np.int64)
        mm = np.concatenate([np.zeros(64, np.int32), np.ones(6, np.int32)])
        o = np.argsort(t, kind="stable")
        slo = [10**7] * 6
        lat, st = ctx.serve(lanes, 6, t[o], mm[o], slo, stats=True)
        assert (lat >= 0).all(), lat
        assert st["h2d_bytes"] > 0 and st["d2h_bytes"] > 0
        # host-ring outputs vs the oracle (request slot s holds input s)
        for m, n in (("lenet5", 32), ("resnet50", 2)):
            yh, per = refs[m]
            got = yh.numpy().reshape(slots[m], per)[:n].astype(np.float64)
            x = synthgen.model_input(m, slots[m])[:n]
            ref = omodels.forward(m, synthgen.weights(m), x)["logits"].reshape(n, -1)
            assert rel_err(got, ref) <= REL_TOL, m
        for gid in (g0, g1):
            ctx.destroy_gpulet(gid)
    finally:
        ctx.close()


def test_serve_chain_spawns_after_completion():
    """gl_serve_chain on a live gpu-let (F3, DESIGN R28): every completed first-stage
    request spawns two second-stage requests that arrive handoff_us after its
    completion; latencies are measured from the application's arrival."""
    import torch
    from paper_2109_01611_b200 import gpulet
    ctx = gpulet.Context(1)
    try:
        mid = ctx.load_model(0, "lenet5", synthgen.weight_file("lenet5"))
        # device buffers first: a whole-GPU executor leaves no SM for torch's fill kernels
        x = torch.zeros(ctx.model_io(mid, 32)[0] // 2, dtype=torch.bfloat16, device="cuda")
        ys = [torch.empty(ctx.model_io(mid, 32)[1] // 4, device="cuda") for _ in range(2)]
        torch.cuda.synchronize()
        (gid, _n), = ctx.create_gpulets(0, [100])
        lanes = [dict(gpulet=gid, model_id=mid, model_slot=s, batch=b, duty_us=200, weight=1, drop_us=0, x=x,
                      y=y) for (s, b), y in zip(((0, 4), (1, 8)), ys)]
        t = (np.arange(20) * 1000).astype(np.int64)
        m = np.zeros(20, np.int32)
        lat, parent, model = ctx.serve_chain(lanes, 2, t, m, [10**7, 10**7], {0: [1, 1]}, 300)
        assert len(lat) == 60 and (lat >= 0).all()
        assert parent[:20].tolist() == [-1] * 20 and model[20:].tolist() == [1] * 40
        assert all(parent[i] == (i - 20) // 2 for i in range(20, 60))    # children of completion order
        for i in range(20, 60):
            assert lat[i] >= lat[parent[i]] + 300
        ctx.destroy_gpulet(gid)
    finally:
        ctx.close()
