"""Write tests/golden/top1_<model>.npz — oracle outputs for the top-1 parity test
(tests/test_gpu_top1.py, north_star "top-1 identical on
>= 99.9 % of samples"): 1,024 LeNet-5 images and 256 requests of every other
model, as batches of 32 drawn by synthgen with batch ids 40, 41, ...

Test infrastructure: calls only synthgen (inputs, weights) and oracle/models.py
(the fp64 forward).  Nothing here comes from the CUDA path.

Stored per model (all float32 unless noted):
  classifiers / BERT : logits [n, classes]
  BERT               : pooled [n, 768] as bf16 bits (uint16; the oracle rounds it to bf16)
  SSD-MobileNet      : per request, the top detection over (prior, class >= 1) of the
                       softmax conf: top_idx (int32, prior * 21 + class), top_val, second_val;
                       and for the first 32 requests every prior's class argmax (uint8)
                       with its top-1 / top-2 gap (float16)

    python scripts/make_top1_golden.py [--models lenet5,...] [--procs 8]
"""
import argparse
import os
import sys

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthgen  # noqa: E402
from oracle import models as omodels  # noqa: E402

N_REQ = {"lenet5": 1024, "googlenet": 256, "resnet50": 256, "ssd_mobilenet_v1": 256, "vgg16": 256, "bert_base": 256}
BATCH = 32
FIRST_BATCH_ID = 40
SSD_ANCHOR_REQS = 32


def _job(args):
    model, batch_id = args
    x = synthgen.model_input(model, BATCH, batch_id)
    return batch_id, omodels.forward(model, synthgen.weights(model), x)


def _bf16_bits(v):
    f = np.asarray(v, np.float64).astype(np.float32)
    return (f.view(np.uint32) >> 16).astype(np.uint16)   # exact: the oracle's pooled values are bf16


def build(model, procs):
    from multiprocessing import Pool
    ids = [FIRST_BATCH_ID + j for j in range(N_REQ[model] // BATCH)]
    with Pool(procs) as pool:
        res = dict(pool.map(_job, [(model, i) for i in ids]))
    outs = [res[i] for i in ids]
    rec = {"batch_ids": np.asarray(ids, np.int32), "batch": np.int32(BATCH)}
    if model == "ssd_mobilenet_v1":
        conf = np.concatenate([o["conf"] for o in outs])              # [n, 3000, 21]
        fg = conf[:, :, 1:].reshape(len(conf), -1)                    # class >= 1
        order = np.argsort(-fg, axis=1, kind="stable")[:, :2]
        top = order[:, 0]
        pr, cl = top // 20, top % 20 + 1
        rec["top_idx"] = (pr * 21 + cl).astype(np.int32)
        rec["top_val"] = np.take_along_axis(fg, order[:, :1], 1)[:, 0].astype(np.float32)
        rec["second_val"] = np.take_along_axis(fg, order[:, 1:2], 1)[:, 0].astype(np.float32)
        a = conf[:SSD_ANCHOR_REQS]
        srt = np.sort(a, axis=-1)
        rec["anchor_top1"] = a.argmax(-1).astype(np.uint8)
        rec["anchor_gap"] = (srt[..., -1] - srt[..., -2]).astype(np.float16)
    else:
        rec["logits"] = np.concatenate([o["logits"] for o in outs]).astype(np.float32)
        if model == "bert_base":
            rec["pooled_bits"] = _bf16_bits(np.concatenate([o["pooled"] for o in outs]))
    path = os.path.join(ROOT, "tests", "golden", f"top1_{model}.npz")
    np.savez_compressed(path, **rec)
    print(path, {k: v.shape for k, v in rec.items()})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default=",".join(synthgen.MODELS))
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    for m in a.models.split(","):
        build(m, a.procs)


if __name__ == "__main__":
    main()
