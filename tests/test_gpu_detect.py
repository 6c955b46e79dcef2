"""F3 parity on a B200: gl_ssd_detect / gl_crop_resize (detect.cu) vs
oracle/detect.py on the same seeded synthetic SSD head outputs and images.
Boxes, scores, classes, priors and counts compare bit for bit (the kernel takes
every integer-deciding step in the precision R27 fixes); crops compare as bf16
bit patterns."""
import numpy as np
import pytest

from oracle import detect as D
from synthgen.gen import f32_to_bf16_bits

pytestmark = pytest.mark.gpu


def heads(n, seed, temp=2.0, quant=0):
    """Seeded synthetic SSD head outputs: loc ~ N(0, 1), conf = softmax(temp * N(0, 1))."""
    rng = np.random.default_rng(seed)
    loc = rng.normal(0, 1, (n, 3000, 4)).astype(np.float32)
    z = temp * rng.normal(0, 1, (n, 3000, 21))
    conf = np.exp(z - z.max(-1, keepdims=True))
    conf = conf / conf.sum(-1, keepdims=True)
    if quant:   # many exactly equal scores: the (score desc, prior asc) order decides
        conf = np.round(conf * quant) / quant
    return loc, conf.astype(np.float32)


def run_gpu(loc, conf, score_thr, iou_thr, top_k, max_det):
    import torch
    from paper_2109_01611_b200 import gpulet
    n = loc.shape[0]
    dl, dc = torch.from_numpy(loc).cuda(), torch.from_numpy(conf).cuda()
    det = torch.full((max(n, 1), max_det, 7), -1.0, device="cuda")
    cnt = torch.full((max(n, 1),), -1, dtype=torch.int32, device="cuda")
    ws = torch.empty(max(gpulet.ssd_detect_workspace(n, top_k), 1), dtype=torch.uint8, device="cuda")
    gpulet.ssd_detect(dl, dc, n, det, cnt, ws, score_thr, iou_thr, top_k, max_det)
    torch.cuda.synchronize()
    return det.cpu().numpy(), cnt.cpu().numpy()


def check(loc, conf, score_thr, iou_thr, top_k, max_det, images=None):
    det, cnt = run_gpu(loc, conf, score_thr, iou_thr, top_k, max_det)
    images = range(loc.shape[0]) if images is None else images
    ref = D.detect(loc[list(images)], conf[list(images)], score_thr, iou_thr, top_k, max_det)
    for r, n in zip(ref, images):
        assert cnt[n] == len(r), (n, cnt[n], len(r))
        want = np.asarray(r, np.float32).reshape(-1, 7)
        np.testing.assert_array_equal(det[n, :len(r)], want)
    return cnt


@pytest.mark.parametrize("seed,score_thr,iou_thr,top_k,max_det", [
    (0, 0.3, 0.45, 200, 100),
    (1, 0.2, 0.5, 64, 37),      # ragged caps
    (2, 0.5, 0.3, 1, 1),        # one candidate per class, one detection
    (3, 0.25, 0.0, 50, 100),    # iou_thr 0: any overlap suppresses
])
def test_detect_vs_oracle(seed, score_thr, iou_thr, top_k, max_det):
    loc, conf = heads(3, seed)
    cnt = check(loc, conf, score_thr, iou_thr, top_k, max_det)
    assert cnt.max() > 0


def test_detect_ties_order_by_prior():
    loc, conf = heads(2, 11, temp=1.0, quant=16)
    check(loc, conf, 0.1, 0.45, 120, 100)


def test_detect_many_candidates_full_sort():
    """score_thr 0: all 3000 priors of every class are candidates (4096-key sort), top_k at its maximum."""
    loc, conf = heads(1, 12, temp=0.5)
    check(loc, conf, 0.0, 0.45, 400, 100)


def test_detect_no_candidates_and_empty_batch():
    loc, conf = heads(2, 13)
    _, cnt = run_gpu(loc, conf, 0.9999, 0.45, 200, 100)
    assert list(cnt) == [0, 0]
    _, cnt = run_gpu(loc[:0], conf[:0], 0.3, 0.45, 200, 100)   # n_img = 0: no-op


def test_detect_bad_args():
    from paper_2109_01611_b200 import gpulet
    with pytest.raises(gpulet.GpuletError):
        gpulet.ssd_detect_workspace(1, 401)
    loc, conf = heads(1, 14)
    with pytest.raises(gpulet.GpuletError):
        run_gpu(loc, conf, 0.3, 0.45, 200, 0)


def test_detect_full_batch_sampled():
    """The traffic workload's SSD batch (32 images) in one launch; three sampled images vs the oracle."""
    loc, conf = heads(32, 21)
    check(loc, conf, 0.3, 0.45, 200, 100, images=[0, 17, 31])


def _crop_case(n, per_img, OH, OW, seed):
    import torch
    from paper_2109_01611_b200 import gpulet
    rng = np.random.default_rng(seed)
    H = W = 300
    img_bits = f32_to_bf16_bits(rng.normal(0, 1, (n, H, W, 8)).astype(np.float32))
    img = img_bits.view(np.uint16)
    loc, conf = heads(n, seed + 1)
    dets = D.detect(loc, conf, 0.3, 0.45, 200, 20)   # the boxes come from the oracle, not the kernel
    max_det = 20
    det = np.zeros((n, max_det, 7), np.float32)
    cnt = np.zeros(n, np.int32)
    for i, r in enumerate(dets):
        r = r[:max(0, per_img - i)]    # fewer detections on later images: zero-filled slots
        cnt[i] = len(r)
        if r:
            det[i, :len(r)] = np.asarray(r, np.float32)
    d_img = torch.from_numpy(img.astype(np.int16)).cuda()
    out = torch.empty((n * per_img, OH, OW, 8), dtype=torch.int16, device="cuda")
    gpulet.crop_resize(d_img, n, H, W, torch.from_numpy(det).cuda(), torch.from_numpy(cnt).cuda(), max_det, per_img,
                       out, OH, OW)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint16)
    imgf = (img.astype(np.uint32) << 16).view(np.float32)
    for i in range(n):
        for k in range(per_img):
            g = got[i * per_img + k]
            if k >= cnt[i]:
                assert not g.any()
                continue
            want = f32_to_bf16_bits(D.crop_resize(imgf[i], det[i, k, :4], OH, OW))
            np.testing.assert_array_equal(g, want)


def test_crop_resize_recogniser_size():
    _crop_case(2, 2, 224, 224, 31)


def test_crop_resize_ragged():
    _crop_case(3, 3, 37, 53, 32)
