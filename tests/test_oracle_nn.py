"""Pins for oracle/nn.py (C1.1 layer definitions) — SURVEY.md §8(c) C1.6.

Each layer is checked against something other than itself: torch-CPU
functional ops (independent library implementation, NCHW), brute-force loops on
tiny shapes, and special cases with closed forms.
"""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import nn


def _rng(s=0):
    return np.random.default_rng(s)


def _brute_conv(x, w, b, s, p):
    N, H, W, C = x.shape
    Co, KH, KW, _ = w.shape
    Ho, Wo = (H + 2 * p - KH) // s + 1, (W + 2 * p - KW) // s + 1
    y = np.zeros((N, Ho, Wo, Co))
    for n, ho, wo, co in itertools.product(range(N), range(Ho), range(Wo), range(Co)):
        acc = b[co]
        for kh, kw, ci in itertools.product(range(KH), range(KW), range(C)):
            hi, wi = ho * s + kh - p, wo * s + kw - p
            if 0 <= hi < H and 0 <= wi < W:
                acc += x[n, hi, wi, ci] * w[co, kh, kw, ci]
        y[n, ho, wo, co] = acc
    return y


@pytest.mark.parametrize("k,s,p", [(1, 1, 0), (3, 1, 1), (3, 2, 1), (5, 1, 2), (7, 2, 3), (1, 2, 0)])
def test_conv_vs_torch(k, s, p):
    r = _rng(k * 10 + s)
    x = r.standard_normal((2, 13, 11, 5))
    w = r.standard_normal((7, k, k, 5))
    b = r.standard_normal(7)
    y = nn.conv2d(x, w, b, s, p)
    t = F.conv2d(torch.tensor(x).permute(0, 3, 1, 2), torch.tensor(w).permute(0, 3, 1, 2),
                 torch.tensor(b), stride=s, padding=p).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(y, t, rtol=1e-10, atol=1e-10)


def test_conv_vs_brute_force():
    r = _rng(1)
    x = r.standard_normal((1, 6, 5, 3))
    w = r.standard_normal((4, 3, 3, 3))
    b = r.standard_normal(4)
    for s, p in [(1, 0), (1, 1), (2, 1), (2, 0)]:
        np.testing.assert_allclose(nn.conv2d(x, w, b, s, p), _brute_conv(x, w, b, s, p), rtol=1e-12)


def test_conv_special_cases():
    r = _rng(2)
    x = r.standard_normal((2, 5, 6, 4))
    # 1x1 conv == matmul over channels
    w = r.standard_normal((3, 1, 1, 4))
    np.testing.assert_allclose(nn.conv2d(x, w, np.zeros(3)), x @ w[:, 0, 0, :].T, rtol=1e-12)
    # delta kernel (centre tap of a 3x3, identity on channels) == identity
    d = np.zeros((4, 3, 3, 4))
    for c in range(4):
        d[c, 1, 1, c] = 1.0
    np.testing.assert_array_equal(nn.conv2d(x, d, np.zeros(4), 1, 1), x)


@pytest.mark.parametrize("s", [1, 2])
def test_dwconv_vs_torch_and_independent_convs(s):
    r = _rng(3 + s)
    x = r.standard_normal((2, 9, 8, 6))
    w = r.standard_normal((6, 3, 3, 1))
    b = r.standard_normal(6)
    y = nn.dwconv2d(x, w, b, s, 1)
    t = F.conv2d(torch.tensor(x).permute(0, 3, 1, 2), torch.tensor(w).permute(0, 3, 1, 2),
                 torch.tensor(b), stride=s, padding=1, groups=6).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(y, t, rtol=1e-10, atol=1e-12)
    # depthwise == C independent single-channel convs
    for c in range(6):
        yc = nn.conv2d(x[..., c:c + 1], w[c:c + 1], b[c:c + 1], s, 1)
        np.testing.assert_allclose(y[..., c:c + 1], yc, rtol=1e-12)


@pytest.mark.parametrize("k,s,p,ceil,H", [(2, 2, 0, False, 28), (3, 2, 1, False, 112),
                                           (3, 2, 0, True, 112), (3, 2, 0, True, 14),
                                           (3, 1, 1, False, 7), (3, 2, 0, True, 13)])
def test_maxpool_vs_torch(k, s, p, ceil, H):
    r = _rng(k + H)
    x = r.standard_normal((2, H, H, 3))
    y = nn.maxpool2d(x, k, s, p, ceil)
    t = F.max_pool2d(torch.tensor(x).permute(0, 3, 1, 2), k, s, p, ceil_mode=ceil).permute(0, 2, 3, 1).numpy()
    np.testing.assert_array_equal(y, t)


def test_googlenet_ceil_mode_sizes():
    # C1.6: GoogLeNet ceil-mode sizes 112 -> 56 -> 28 -> 14 -> 7
    sizes = [112]
    for _ in range(4):
        sizes.append(nn.pool_out_size(sizes[-1], 3, 2, 0, True))
    assert sizes == [112, 56, 28, 14, 7]


def test_layernorm_gelu_softmax():
    r = _rng(5)
    x = r.standard_normal((4, 768)) * 3 + 1
    g, b = r.standard_normal(768), r.standard_normal(768)
    t = F.layer_norm(torch.tensor(x), (768,), torch.tensor(g), torch.tensor(b), eps=1e-12).numpy()
    np.testing.assert_allclose(nn.layernorm(x, g, b), t, rtol=1e-9, atol=1e-9)
    z = nn.layernorm(x, np.ones(768), np.zeros(768))
    np.testing.assert_allclose(z.mean(-1), 0, atol=1e-12)
    np.testing.assert_allclose(z.var(-1), 1, rtol=1e-9)
    np.testing.assert_allclose(nn.gelu(x), F.gelu(torch.tensor(x)).numpy(), rtol=1e-12, atol=1e-14)
    assert nn.gelu(np.array([0.0]))[0] == 0.0
    sm = nn.softmax(x)
    np.testing.assert_allclose(sm.sum(-1), 1, rtol=1e-12)
    np.testing.assert_allclose(sm, torch.softmax(torch.tensor(x), -1).numpy(), rtol=1e-12)
    # shift invariance (max-subtraction must not change the value)
    np.testing.assert_allclose(nn.softmax(x + 100.0), sm, rtol=1e-10)


def test_rbf16_matches_torch():
    r = _rng(6)
    x = np.concatenate([r.standard_normal(10000) * 10, r.standard_normal(1000) * 1e-3,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.005859375])])
    t = torch.tensor(x, dtype=torch.float64).to(torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    np.testing.assert_array_equal(nn.rbf16(x), t)


def test_linear_and_avgpool():
    r = _rng(7)
    x, w, b = r.standard_normal((3, 5)), r.standard_normal((4, 5)), r.standard_normal(4)
    np.testing.assert_allclose(nn.linear(x, w, b), F.linear(torch.tensor(x), torch.tensor(w), torch.tensor(b)).numpy())
    y = r.standard_normal((2, 7, 7, 3))
    np.testing.assert_allclose(nn.global_avgpool(y), F.adaptive_avg_pool2d(torch.tensor(y).permute(0, 3, 1, 2), 1)[..., 0, 0].numpy())
