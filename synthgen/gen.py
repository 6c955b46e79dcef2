"""Seeded generators (numpy PCG64) for weights and inputs — SURVEY.md §8(c) C1.3.

Seeds: weights 1000 + model index (canonical order le, goo, res, ssd, vgg, bert);
inputs 2000 + model index + 100 * batch_id.  Values are drawn in fp32/fp64,
then rounded to bf16 (round-to-nearest-even) because bf16 is the storage and
operand type of both the CUDA path and the oracle (C1.4).  Encoding values as
bf16 bit patterns is storage, not the method's arithmetic.
"""
import os
import numpy as np

from .manifest import MODELS, MODEL_INDEX, manifest, input_shape, BERT_SEQ, BERT_VOCAB

_CACHE = os.environ.get("GPULET_WEIGHT_CACHE", "/tmp/gpulet_weights")


def f32_to_bf16_bits(x):
    """fp32 -> bf16 bit patterns (uint16), round-to-nearest-even (finite inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def bf16_bits_to_f32(b):
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _draw(rng, shape, kind):
    n = int(np.prod(shape))
    if kind in ("he", "he_q"):
        fan_in = int(np.prod(shape[1:]))
        v = rng.standard_normal(n, dtype=np.float32) * np.float32(np.sqrt(2.0 / fan_in))
        if kind == "he_q":
            v *= np.float32(0.25)
    elif kind == "bias":
        v = rng.uniform(-0.05, 0.05, n).astype(np.float32)
    elif kind == "bert":
        v = rng.standard_normal(n, dtype=np.float32) * np.float32(0.02)
    elif kind == "ones":
        v = np.ones(n, np.float32)
    elif kind == "zeros":
        v = np.zeros(n, np.float32)
    else:
        raise ValueError(kind)
    return f32_to_bf16_bits(v).reshape(shape)


def weights(model):
    """{name: uint16 bf16 bits array} drawn in manifest order from PCG64(1000+idx)."""
    rng = np.random.Generator(np.random.PCG64(1000 + MODEL_INDEX[model]))
    return {name: _draw(rng, shape, kind) for name, shape, kind in manifest(model)}


def weight_file(model, directory=None):
    """Write (once) and return the path of the model's GLW1 weight file.

    Format (read by the C-ABI `gl_load_model`): first line "GLW1 <header_bytes>";
    then one line per parameter "name bf16 ndim d0 .. offset nbytes"; "END".
    The header is zero-padded to header_bytes (a multiple of 4096); offsets are
    relative to the end of the header, each 256-byte aligned; data little-endian.
    """
    directory = directory or _CACHE
    os.makedirs(directory, exist_ok=True)
    path = os.path.join(directory, f"{model}.glw")
    if os.path.exists(path):
        return path
    w = weights(model)
    lines, off = [], 0
    for name, shape, _k in manifest(model):
        nbytes = int(np.prod(shape)) * 2
        lines.append(f"{name} bf16 {len(shape)} {' '.join(map(str, shape))} {off} {nbytes}")
        off += (nbytes + 255) // 256 * 256
    body = ("\n".join(lines) + "\nEND\n").encode()
    first = b"GLW1 %d\n"
    hdr_len = 4096
    while len(first % hdr_len) + len(body) > hdr_len:
        hdr_len += 4096
    header = (first % hdr_len) + body
    header += b"\0" * (hdr_len - len(header))
    tmp = path + f".tmp{os.getpid()}"
    with open(tmp, "wb") as f:
        f.write(header)
        pos = 0
        for name, shape, _k in manifest(model):
            data = w[name].astype("<u2").tobytes()
            f.write(data)
            pos += len(data)
            pad = (len(data) + 255) // 256 * 256 - len(data)
            f.write(b"\0" * pad)
    os.replace(tmp, path)
    return path


def _input_rng(model, batch_id):
    return np.random.Generator(np.random.PCG64(2000 + MODEL_INDEX[model] + 100 * batch_id))


def image_batch(model, batch, batch_id=0):
    """ImageNet-normalised-like NHWC image batch: N(0,1) clipped to +-3, bf16 bits."""
    shape = input_shape(model, batch)
    rng = _input_rng(model, batch_id)
    x = np.clip(rng.standard_normal(shape, dtype=np.float32), -3.0, 3.0)
    return f32_to_bf16_bits(x)


def mnist_batch(batch, batch_id=0):
    """MNIST-like [b,28,28,1]: 80 % zeros, 20 % U(0,1); bf16 bits."""
    rng = _input_rng("lenet5", batch_id)
    shape = (batch, 28, 28, 1)
    keep = rng.random(shape) >= 0.8
    v = rng.random(shape).astype(np.float32)
    return f32_to_bf16_bits(np.where(keep, v, np.float32(0)))


def bert_ids(batch, batch_id=0):
    """int32 [b,128]: [CLS]=101 at 0, [SEP]=102 at 127, rest uniform in [1000, 30522)."""
    rng = _input_rng("bert_base", batch_id)
    ids = rng.integers(1000, BERT_VOCAB, size=(batch, BERT_SEQ), dtype=np.int64)
    ids[:, 0] = 101
    ids[:, -1] = 102
    return ids.astype(np.int32)


def model_input(model, batch, batch_id=0):
    if model == "lenet5":
        return mnist_batch(batch, batch_id)
    if model == "bert_base":
        return bert_ids(batch, batch_id)
    return image_batch(model, batch, batch_id)


def pad_channels(x_bits, c=8):
    """NHWC bf16 bits [..., C] -> [..., c] with zero channels (GPU input layout)."""
    out = np.zeros(x_bits.shape[:-1] + (c,), np.uint16)
    out[..., : x_bits.shape[-1]] = x_bits
    return out
