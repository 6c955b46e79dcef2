"""Pins for oracle/models.py (C1.2 topologies) — closed-form totals and invariants.

The topologies are readings (C6 #1-#4, parity unpinned as topologies), but
their totals are fixed by the published architectures:
  LeNet-5 61,706 params; ResNet-50 4.09 GMAC / 25.5 M params;
  VGG-16 15.47 GMAC / 138.4 M params; BERT-base 109.5 M params
  (+ 2-class head), 11.17 GMAC at L=128; SSD 3,000 priors.
"""
import numpy as np
import pytest

import synthgen
from oracle import models, nn


def _params(m):
    return sum(int(np.prod(s)) for _n, s, _k in synthgen.manifest(m))


def test_param_counts():
    assert _params("lenet5") == 61706
    assert abs(_params("resnet50") / 1e6 - 25.53) < 0.02
    assert abs(_params("vgg16") / 1e6 - 138.36) < 0.01
    assert abs(_params("bert_base") / 1e6 - 109.48) < 0.02
    assert abs(_params("googlenet") / 1e6 - 7.0) < 0.05


@pytest.mark.parametrize("m,gmac,tol", [("resnet50", 4.089, 0.005), ("googlenet", 1.583, 0.005),
                                        ("ssd_mobilenet_v1", 1.527, 0.005), ("lenet5", 0.000417, 2e-6)])
def test_mac_totals(m, gmac, tol):
    w = synthgen.weights(m)
    _out, macs = models.forward(m, w, synthgen.model_input(m, 1), return_macs=True)
    assert abs(macs / 1e9 - gmac) < tol


@pytest.mark.slow
def test_mac_totals_large():
    for m, gmac in [("vgg16", 15.470), ("bert_base", 11.174)]:
        w = synthgen.weights(m)
        _out, macs = models.forward(m, w, synthgen.model_input(m, 1), return_macs=True)
        assert abs(macs / 1e9 - gmac) < 0.005, (m, macs)


def test_lenet_batch_consistency_and_shapes():
    w = synthgen.weights("lenet5")
    x = synthgen.mnist_batch(4)
    y = models.forward("lenet5", w, x)["logits"]
    assert y.shape == (4, 10)
    # per-sample independence: row i of a batch == the forward of sample i alone
    for i in range(4):
        yi = models.forward("lenet5", w, x[i:i + 1])["logits"]
        np.testing.assert_array_equal(y[i:i + 1], yi)


def test_ssd_priors_and_softmax():
    w = synthgen.weights("ssd_mobilenet_v1")
    out = models.forward("ssd_mobilenet_v1", w, synthgen.model_input("ssd_mobilenet_v1", 1))
    assert out["loc"].shape == (1, 3000, 4)
    assert out["conf"].shape == (1, 3000, 21)
    np.testing.assert_allclose(out["conf"].sum(-1), 1.0, rtol=1e-6)


def test_rounding_points_are_bf16():
    """Intermediate activations are bf16-exact (C1.4): rbf16 is idempotent on them."""
    w = synthgen.weights("lenet5")
    P = models._W(w)
    x = nn.bits_to_f64(synthgen.mnist_batch(2))
    h = nn.rbf16(nn.relu(P.conv(x, "conv1", 1, 2)))
    np.testing.assert_array_equal(nn.rbf16(h), h)
