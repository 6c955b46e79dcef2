"""Model parity on a B200: every model's forward through the C-ABI (gpu-let
executor, submit/poll) vs the oracle forward (oracle/models.py) on the same
seeded inputs and weights (synthgen).  Bars (north_star): max relative error
<= 2e-2 on the final outputs, top-1 identical on >= 99.9 % of unambiguous samples."""
import numpy as np
import pytest

import synthgen
from oracle import models as omodels
from tests.gpu_util import (REL_TOL, TOP1_TOL, bert_logit_bound, rel_err, split_outputs, to_dev_bf16,
                            top1_agreement)

pytestmark = pytest.mark.gpu

BATCH = {"lenet5": 32, "googlenet": 3, "resnet50": 3, "ssd_mobilenet_v1": 2, "vgg16": 2, "bert_base": 2}


@pytest.fixture(scope="module")
def served():
    from paper_2109_01611_b200 import gpulet
    c = gpulet.Context(1)
    mids = {m: c.load_model(0, m, synthgen.weight_file(m)) for m in synthgen.MODELS}
    gid, nsm = c.create_gpulet(0, 100)
    yield c, mids, gid
    c.close()


def _device_input(model, batch, batch_id=0):
    import torch
    x = synthgen.model_input(model, batch, batch_id)
    if model == "bert_base":
        return x, torch.from_numpy(x).cuda()
    xd = synthgen.pad_channels(x, 8) if model != "lenet5" else x
    return x, to_dev_bf16(xd)


def run_model(c, gid, mid, model, batch, batch_id=0):
    import torch
    x, xd = _device_input(model, batch, batch_id)
    _inb, outb = c.model_io(mid, batch)
    y = torch.empty(outb // 4, dtype=torch.float32, device="cuda")
    t = c.submit_batch(gid, mid, xd, y, batch, 100.0)
    comp = c.wait(t)
    return x, y.cpu().numpy(), comp


@pytest.mark.parametrize("model", synthgen.MODELS)
def test_model_parity(served, model):
    c, mids, gid = served
    b = BATCH[model]
    x, got, comp = run_model(c, gid, mids[model], model, b)
    assert comp.t_end_ns > comp.t_start_ns
    ref = omodels.forward(model, synthgen.weights(model), x)
    out = split_outputs(model, got, b)
    if model == "ssd_mobilenet_v1":
        assert rel_err(out["loc"], ref["loc"]) <= REL_TOL
        assert rel_err(out["conf"], ref["conf"]) <= REL_TOL
        err = np.abs(out["conf"] - ref["conf"]).max()
        strict, judged, amb = top1_agreement(out["conf"], ref["conf"], 4 * err)
        assert judged >= TOP1_TOL, (strict, judged, amb)
    else:
        ref_l, got_l = ref["logits"], out["logits"].reshape(ref["logits"].shape)
        if model == "bert_base":   # R30
            assert (np.abs(got_l - ref_l) <= bert_logit_bound(ref["pooled"])).all()
        else:
            e = rel_err(got_l, ref_l)
            assert e <= REL_TOL, e
        err = np.abs(got_l - ref_l).max()
        strict, judged, amb = top1_agreement(got_l, ref_l, 4 * err)
        assert judged >= TOP1_TOL, (strict, judged, amb)
        if model == "bert_base":   # the 768-d pooled [CLS] representation, element by element
            assert rel_err(out["pooled"], ref["pooled"]) <= REL_TOL


def test_batch_sizes_ragged(served):
    """Batch 1 and 5 (ragged M tails) give the same per-sample outputs as the oracle."""
    c, mids, gid = served
    for b in (1, 5):
        x, got, _ = run_model(c, gid, mids["resnet50"], "resnet50", b, batch_id=3)
        ref = omodels.forward("resnet50", synthgen.weights("resnet50"), x)["logits"]
        assert rel_err(split_outputs("resnet50", got, b)["logits"], ref) <= REL_TOL
