"""F3 SSD post-processing and crop stage of the `traffic` pipeline (ORACLE —
test infrastructure only; imported by tests/, smoke() and bench's reference
legs, never by the product path).

PAPER.md names the application only ("traffic" = SSD-MobileNet
object detection whose detected objects go to GoogLeNet and VGG-16
recognisers); it says nothing about box decoding, NMS or cropping (SURVEY C6
#3).  This module is therefore the textbook SSD detector output stage, with
the readings listed in DESIGN.md §2 R27:

  priors   6 per location on the six maps 19,10,5,3,2,1 (our topology,
           oracle/models.py ssd_mobilenet_v1), order (h, w, prior) like the
           heads; scale s_k = 0.2 + 0.75 k / 5 (k = 0..5), s_6 = 1; priors
           0..4 have aspect ratios 1, 2, 1/2, 3, 1/3 at s_k (w = s sqrt(a),
           h = s / sqrt(a)), prior 5 has ratio 1 at sqrt(s_k s_{k+1});
           centres ((j + .5)/f, (i + .5)/f).  Computed in fp64, stored fp32.
  decode   variances (0.1, 0.2): cx = pcx + l0 0.1 pw, cy = pcy + l1 0.1 ph,
           w = pw exp(0.2 l2), h = ph exp(0.2 l3), corners cx -/+ w/2, in
           fp64 (each product/sum rounded separately, no FMA), rounded to
           fp32, then clipped to [0, 1].
  select   per class c = 1..20 (0 = background): priors with conf > score_thr
           (fp32 compare), ordered by (score desc, prior asc), first top_k.
  NMS      greedy (Neubeck & Van Gool): walk the ordered candidates, keep one
           unless its IoU with an already kept box of the class is > iou_thr.
           IoU in fp32: inter = max(0, min(x2) - max(x1)) * max(0, min(y2) -
           max(y1)), union = area_a + area_b - inter, IoU = inter / union (a
           0/0 is NaN and never suppresses).
  merge    all classes' kept boxes of an image ordered by (score desc, class
           asc, prior asc), first max_det.
  crop     each detection's box, in the 300 x 300 input, resized to 224 x 224
           by bilinear sampling with half-pixel centres (align_corners=False):
           source x = x1 W + (ox + .5) (x2 - x1) W / OW - .5, clamped to
           [0, W - 1], fp32; output rounded to bf16 (the recogniser's input).

Parity status: priors pinned by closed-form facts (count, map-1 centre,
sizes), decode by the encode/decode round trip, NMS against
torchvision.ops.nms and brute-force invariants, crop against
torch.nn.functional.interpolate on full-image boxes and exact linear ramps
(tests/test_oracle_detect.py).
"""
import math

import numpy as np

MAPS = (19, 10, 5, 3, 2, 1)
N_PRIORS = 3000
N_CLASSES = 21
VAR_XY, VAR_WH = 0.1, 0.2


def scales():
    """s_k = s_min + (s_max - s_min) k / (m - 1), s_min 0.2, s_max 0.95, m 6; s_6 = 1."""
    return [0.2 + 0.75 * k / 5.0 for k in range(6)] + [1.0]


def priors():
    """[3000, 4] fp32 (cx, cy, w, h), in head order (map, h, w, prior)."""
    s = scales()
    out = []
    for k, f in enumerate(MAPS):
        for i in range(f):
            for j in range(f):
                cx, cy = (j + 0.5) / f, (i + 0.5) / f
                for a in (1.0, 2.0, 0.5, 3.0, 1.0 / 3.0):
                    r = math.sqrt(a)
                    out.append((cx, cy, s[k] * r, s[k] / r))
                sp = math.sqrt(s[k] * s[k + 1])
                out.append((cx, cy, sp, sp))
    P = np.asarray(out, np.float64).astype(np.float32)
    assert P.shape == (N_PRIORS, 4)
    return P


def decode(loc, P):
    """loc [..., 4] fp32, P [3000, 4] fp32 -> boxes [..., 4] fp32 (x1, y1, x2, y2) in [0, 1]."""
    l = loc.astype(np.float64)
    p = P.astype(np.float64)
    pcx, pcy, pw, ph = p[..., 0], p[..., 1], p[..., 2], p[..., 3]
    cx = pcx + (l[..., 0] * VAR_XY) * pw
    cy = pcy + (l[..., 1] * VAR_XY) * ph
    w = pw * np.exp(l[..., 2] * VAR_WH)
    h = ph * np.exp(l[..., 3] * VAR_WH)
    b = np.stack([cx - w * 0.5, cy - h * 0.5, cx + w * 0.5, cy + h * 0.5], axis=-1).astype(np.float32)
    return np.clip(b, np.float32(0.0), np.float32(1.0))


def iou(a, b):
    """fp32 IoU of two boxes (x1, y1, x2, y2), the order of operations above."""
    f = np.float32
    with np.errstate(invalid="ignore", divide="ignore"):
        iw = max(f(0), f(min(a[2], b[2]) - max(a[0], b[0])))
        ih = max(f(0), f(min(a[3], b[3]) - max(a[1], b[1])))
        inter = f(iw * ih)
        area_a = f(f(a[2] - a[0]) * f(a[3] - a[1]))
        area_b = f(f(b[2] - b[0]) * f(b[3] - b[1]))
        union = f(f(area_a + area_b) - inter)
        return f(inter / union)


def nms_class(boxes, scores, score_thr, iou_thr, top_k):
    """One image, one class: kept prior indices in (score desc, prior asc) order."""
    cand = [i for i in range(len(scores)) if scores[i] > np.float32(score_thr)]
    cand.sort(key=lambda i: (-float(scores[i]), i))
    cand = cand[:top_k]
    kept = []
    for i in cand:
        if all(not (iou(boxes[i], boxes[k]) > np.float32(iou_thr)) for k in kept):
            kept.append(i)
    return kept


def detect(loc, conf, score_thr=0.05, iou_thr=0.45, top_k=200, max_det=100):
    """loc [n, 3000, 4], conf [n, 3000, 21] fp32 -> list per image of
    detections (x1, y1, x2, y2, score, class, prior)."""
    P = priors()
    out = []
    for n in range(loc.shape[0]):
        boxes = decode(loc[n], P)
        dets = []
        for c in range(1, N_CLASSES):
            s = conf[n, :, c].astype(np.float32)
            for i in nms_class(boxes, s, score_thr, iou_thr, top_k):
                dets.append((float(s[i]), c, i))
        dets.sort(key=lambda d: (-d[0], d[1], d[2]))
        out.append([tuple(float(v) for v in boxes[i]) + (sc, c, i) for sc, c, i in dets[:max_det]])
    return out


def crop_resize(img, box, OH=224, OW=224):
    """img [H, W, C] fp32 (bf16 values), box (x1, y1, x2, y2) in [0, 1] ->
    [OH, OW, C] fp32 rounded to bf16 by the caller.  Plain per-pixel loops
    over the bilinear formula (fp32 arithmetic as stated above)."""
    f = np.float32
    H, W, C = img.shape
    x1, y1, x2, y2 = (f(v) for v in box)
    sw = f(f(f(x2 - x1) * f(W)) / f(OW))
    sh = f(f(f(y2 - y1) * f(H)) / f(OH))
    out = np.zeros((OH, OW, C), np.float32)
    for oy in range(OH):
        sy = f(f(f(y1 * f(H)) + f(f(f(oy) + f(0.5)) * sh)) - f(0.5))
        sy = min(max(sy, f(0)), f(H - 1))
        y0 = int(math.floor(sy))
        y1i = min(y0 + 1, H - 1)
        wy = f(sy - f(y0))
        for ox in range(OW):
            sx = f(f(f(x1 * f(W)) + f(f(f(ox) + f(0.5)) * sw)) - f(0.5))
            sx = min(max(sx, f(0)), f(W - 1))
            x0 = int(math.floor(sx))
            x1i = min(x0 + 1, W - 1)
            wx = f(sx - f(x0))
            top = img[y0, x0] + (img[y0, x1i] - img[y0, x0]) * wx
            bot = img[y1i, x0] + (img[y1i, x1i] - img[y1i, x0]) * wx
            out[oy, ox] = top + (bot - top) * wy
    return out
