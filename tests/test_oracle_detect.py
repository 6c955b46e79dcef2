"""Pins for oracle/detect.py (F3: SSD post-processing + crops; R27).
Each pin checks the oracle against something other than itself: closed-form
facts of the prior layout, the inverse of the decode (SSD box encoding),
torchvision's NMS, brute-force invariants of greedy NMS, and
torch.nn.functional.interpolate / exact linear ramps for the crop."""
import math

import numpy as np
import pytest

from oracle import detect as D


def test_priors_closed_form():
    P = D.priors()
    assert P.shape == (3000, 4)
    # 6 per location over 19^2 + 10^2 + 5^2 + 3^2 + 2^2 + 1 locations
    assert 6 * sum(f * f for f in D.MAPS) == 3000
    # first prior: map 19, cell (0, 0), ratio 1 at s_0 = 0.2
    np.testing.assert_allclose(P[0], [0.5 / 19, 0.5 / 19, 0.2, 0.2], rtol=1e-6)
    # ratio 2 prior: w/h = 2, w*h = s^2
    assert abs(P[1, 2] / P[1, 3] - 2) < 1e-5 and abs(P[1, 2] * P[1, 3] - 0.04) < 1e-6
    # last map (1x1): centre (0.5, 0.5); prior 0 side 0.95, prior 5 side sqrt(0.95 * 1)
    np.testing.assert_allclose(P[-6, :2], [0.5, 0.5])
    np.testing.assert_allclose(P[-6, 2], 0.95, rtol=1e-6)
    np.testing.assert_allclose(P[-1, 2], math.sqrt(0.95), rtol=1e-6)
    # map 10 starts after 19*19*6 priors, its scale is 0.35
    np.testing.assert_allclose(P[19 * 19 * 6, 2], 0.35, rtol=1e-6)


def test_decode_inverts_ssd_encoding():
    """Encode known boxes (the SSD regression target, written independently as
    the inverse map) and decode them back."""
    rng = np.random.default_rng(3)
    P = D.priors().astype(np.float64)
    gt_c = rng.uniform(0.3, 0.7, (3000, 2))
    gt_wh = rng.uniform(0.05, 0.3, (3000, 2))
    loc = np.empty((3000, 4))
    loc[:, 0] = (gt_c[:, 0] - P[:, 0]) / (P[:, 2] * 0.1)
    loc[:, 1] = (gt_c[:, 1] - P[:, 1]) / (P[:, 3] * 0.1)
    loc[:, 2] = np.log(gt_wh[:, 0] / P[:, 2]) / 0.2
    loc[:, 3] = np.log(gt_wh[:, 1] / P[:, 3]) / 0.2
    b = D.decode(loc.astype(np.float32), D.priors())
    want = np.concatenate([gt_c - gt_wh / 2, gt_c + gt_wh / 2], axis=1)
    np.testing.assert_allclose(b, want, atol=2e-5)
    # clipping: a huge box becomes the unit square
    big = D.decode(np.array([[0, 0, 30, 30]], np.float32), D.priors()[:1])
    np.testing.assert_array_equal(big[0], [0, 0, 1, 1])


def _rand_boxes(rng, n):
    c = rng.uniform(0.2, 0.8, (n, 2))
    wh = rng.uniform(0.05, 0.4, (n, 2))
    return np.concatenate([c - wh / 2, c + wh / 2], axis=1).astype(np.float32)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_nms_matches_torchvision(seed):
    torch = pytest.importorskip("torch")
    tvops = pytest.importorskip("torchvision.ops")
    rng = np.random.default_rng(seed)
    n = 300
    boxes = _rand_boxes(rng, n)
    scores = rng.permutation(n).astype(np.float32) / n + 0.01   # distinct scores
    mine = D.nms_class(boxes, scores, 0.0, 0.45, n)
    ref = tvops.nms(torch.from_numpy(boxes).double(), torch.from_numpy(scores).double(), 0.45).tolist()
    assert mine == ref


def test_nms_invariants_and_topk():
    rng = np.random.default_rng(7)
    boxes = _rand_boxes(rng, 120)
    scores = np.round(rng.uniform(0, 1, 120), 2).astype(np.float32)   # many ties
    kept = D.nms_class(boxes, scores, 0.3, 0.5, 50)
    cand = sorted([i for i in range(120) if scores[i] > np.float32(0.3)], key=lambda i: (-scores[i], i))[:50]
    # kept is an ordered subsequence of the candidates
    it = iter(cand)
    assert all(k in it for k in kept)
    # no two kept boxes overlap more than the threshold
    for a in range(len(kept)):
        for b in range(a + 1, len(kept)):
            assert not D.iou(boxes[kept[a]], boxes[kept[b]]) > 0.5
    # each dropped candidate overlaps an earlier kept box above the threshold
    for i in cand:
        if i not in kept:
            pos = cand.index(i)
            assert any(D.iou(boxes[i], boxes[k]) > 0.5 for k in kept if cand.index(k) < pos)


def test_iou_closed_forms():
    f = np.float32
    a = np.array([0, 0, 1, 1], np.float32)
    assert D.iou(a, a) == f(1)
    assert D.iou(a, np.array([0.5, 0, 1.5, 1], np.float32)) == f(0.5) / f(1.5)
    assert D.iou(a, np.array([2, 2, 3, 3], np.float32)) == 0
    assert np.isnan(D.iou(np.zeros(4, np.float32), np.zeros(4, np.float32)))


def test_detect_merge_order_and_caps():
    rng = np.random.default_rng(5)
    loc = rng.normal(0, 1, (2, 3000, 4)).astype(np.float32)
    logits = rng.normal(0, 2, (2, 3000, 21))
    conf = (np.exp(logits) / np.exp(logits).sum(-1, keepdims=True)).astype(np.float32)
    dets = D.detect(loc, conf, score_thr=0.3, iou_thr=0.45, top_k=50, max_det=40)
    for img in dets:
        assert 0 < len(img) <= 40
        keys = [(-d[4], d[5], d[6]) for d in img]
        assert keys == sorted(keys)
        assert all(1 <= d[5] <= 20 and d[4] > np.float32(0.3) for d in img)
        assert all(0 <= v <= 1 for d in img for v in d[:4])


def test_crop_full_box_is_interpolate():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(1)
    img = rng.normal(0, 1, (30, 30, 3)).astype(np.float32)
    got = D.crop_resize(img, (0, 0, 1, 1), 22, 22)
    ref = torch.nn.functional.interpolate(torch.from_numpy(img).permute(2, 0, 1)[None], size=(22, 22),
                                          mode="bilinear", align_corners=False)[0].permute(1, 2, 0).numpy()
    np.testing.assert_allclose(got, ref, atol=1e-5)


def test_crop_linear_ramp_exact():
    """Bilinear sampling reproduces a linear function inside the image."""
    H = W = 40
    yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    img = np.stack([xx, yy, 2 * xx + 3 * yy], axis=-1).astype(np.float32)
    box = (0.25, 0.2, 0.75, 0.6)
    got = D.crop_resize(img, box, 16, 16)
    ox = np.arange(16)
    sx = 0.25 * W + (ox + 0.5) * (0.5 * W / 16) - 0.5
    sy = 0.2 * H + (ox + 0.5) * (0.4 * H / 16) - 0.5
    np.testing.assert_allclose(got[0, :, 0], sx, atol=1e-4)
    np.testing.assert_allclose(got[:, 0, 1], sy, atol=1e-4)
    np.testing.assert_allclose(got[..., 2], 2 * got[..., 0] + 3 * got[..., 1], atol=1e-3)
