"""Helpers shared by the -m gpu tests (test infrastructure)."""
import numpy as np

REL_TOL = 2e-2          # north_star: max relative error <= 2e-2 (bf16 operands, fp32 accumulation)
TOP1_TOL = 0.999        # north_star: top-1 identical on >= 99.9 % of (unambiguous) samples


def to_dev_bf16(bits):
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).cuda()


def from_dev_bf16(t):
    import torch
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def bits_to_f64(bits):
    return (np.ascontiguousarray(bits, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def rel_err(got, ref):
    ref = np.asarray(ref, np.float64)
    got = np.asarray(got, np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def top1_agreement(got, ref, tau):
    """(strict, judged, ambiguous_fraction): judged excludes samples whose oracle
    top-1/top-2 gap is <= tau."""
    ref = np.asarray(ref).reshape(-1, ref.shape[-1])
    got = np.asarray(got).reshape(-1, got.shape[-1])
    a, b = ref.argmax(-1), got.argmax(-1)
    strict = float((a == b).mean())
    srt = np.sort(ref, axis=-1)
    gap = srt[:, -1] - srt[:, -2]
    keep = gap > tau
    judged = float((a[keep] == b[keep]).mean()) if keep.any() else 1.0
    return strict, judged, float(1 - keep.mean())


def split_outputs(model, y, b):
    """The GPU output buffer of one batch (fp32 view, gl_model_io layout) as the
    oracle's output dict: logits [b,classes]; SSD loc/conf; BERT logits and the
    bf16 pooled [CLS] vector at byte offset roundup(8b, 16)."""
    y = np.asarray(y)
    if model == "ssd_mobilenet_v1":
        yf = y.astype(np.float64)
        return {"loc": yf[: b * 3000 * 4].reshape(b, 3000, 4),
                "conf": yf[b * 3000 * 4: b * 3000 * 25].reshape(b, 3000, 21)}
    if model == "bert_base":
        y32 = np.ascontiguousarray(y, np.float32)
        off = (b * 8 + 15) // 16 * 16
        pooled = bits_to_f64(y32.view(np.uint16)[off // 2: off // 2 + b * 768]).reshape(b, 768)
        return {"logits": y32[: 2 * b].astype(np.float64).reshape(b, 2), "pooled": pooled}
    return {"logits": np.asarray(y, np.float64).reshape(b, -1)}


def bert_logit_bound(pooled_ref):
    """Per-element tolerance of BERT's 2 logits (DESIGN R30): REL_TOL times the
    magnitude of the terms the logit sums, sum_k |pooled_k W_ck| (+ |b_c|).  The
    logits (|l| ~ 0.2) are a near-cancelling sum of terms ~30x larger, so a
    relative bound on the logits themselves measures the cancellation, not the
    kernels; the pooled vector they come from is checked at REL_TOL as is."""
    import synthgen
    w = synthgen.weights("bert_base")
    W, b = bits_to_f64(w["cls.w"]), bits_to_f64(w["cls.b"])
    return REL_TOL * (np.abs(np.asarray(pooled_ref, np.float64)) @ np.abs(W).T + np.abs(b))
