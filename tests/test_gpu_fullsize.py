"""Parity at the bench's full sizes (BASELINE configs: batch 32 on partial
gpu-lets, the launch configuration bench.py serves): each model's batch-32
forward on an 80 % gpu-let, checked on sampled images (first, a middle one,
last) against the oracle run on those images alone (per-image outputs do not
depend on the batch), plus a ResNet-50 sweep over the gpu-let grid (cfg2) on
a ragged batch."""
import numpy as np
import pytest

import synthgen
from oracle import models as omodels
from tests.gpu_util import REL_TOL, bert_logit_bound, rel_err, split_outputs

pytestmark = pytest.mark.gpu

SAMPLE = {"googlenet": (0, 31), "resnet50": (0, 17, 31), "ssd_mobilenet_v1": (0, 31), "vgg16": (31,),
          "bert_base": (0, 31)}


@pytest.fixture(scope="module")
def ctx():
    from paper_2109_01611_b200 import gpulet
    c = gpulet.Context(1)
    c.mids = {m: c.load_model(0, m, synthgen.weight_file(m)) for m in synthgen.MODELS}
    yield c
    c.close()


def _run(c, gid, m, b, batch_id):
    import torch
    from tools import common
    xd = common.device_input(m, b, batch_id)
    y = torch.empty(c.model_io(c.mids[m], b)[1] // 4, device="cuda")
    c.wait(c.submit_batch(gid, c.mids[m], xd, y, b, 100.0))
    return y.cpu().numpy()


def _check(m, got, b, idx, batch_id):
    x = synthgen.model_input(m, b, batch_id)[list(idx)]
    ref = omodels.forward(m, synthgen.weights(m), x)
    out = split_outputs(m, got, b)
    for k in ref:
        mine = out[k][list(idx)]
        if m == "bert_base" and k == "logits":   # R30
            assert (np.abs(mine - ref[k].reshape(mine.shape)) <= bert_logit_bound(ref["pooled"])).all()
        else:
            assert rel_err(mine, ref[k].reshape(mine.shape)) <= REL_TOL, (m, k)


@pytest.mark.parametrize("m", ["googlenet", "resnet50", "ssd_mobilenet_v1", "vgg16", "bert_base"])
def test_batch32_on_80pct_gpulet_sampled(ctx, m):
    (gid, nsm), = ctx.create_gpulets(0, [80])
    try:
        assert nsm < 148
        got = _run(ctx, gid, m, 32, batch_id=5)
        _check(m, got, 32, SAMPLE[m], 5)
    finally:
        ctx.destroy_gpulet(gid)


@pytest.mark.parametrize("pct", [20, 40, 50, 60, 100])
def test_resnet50_grid_ragged(ctx, pct):
    (gid, _nsm), = ctx.create_gpulets(0, [pct])
    try:
        got = _run(ctx, gid, "resnet50", 13, batch_id=7)
        _check("resnet50", got, 13, (0, 12), 7)
    finally:
        ctx.destroy_gpulet(gid)
