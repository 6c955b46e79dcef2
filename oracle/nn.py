"""C1.1 layer definitions (ORACLE — test infrastructure only).

Plain definitions of the layers the six models use,
NHWC, float64 accumulation.  Values fed in are bf16-exact; `rbf16` rounds a
result to bf16 at the points C1.4 fixes (the paper states no precision, D4;
the north_star fixes "bf16 inputs with fp32 accumulation").

Every function is pinned in tests/test_oracle_nn.py against torch-CPU
functional ops and brute-force loops on tiny shapes.
"""
import numpy as np
from scipy.special import erf


def rbf16(x):
    """Round to bf16 (RNE) via fp32, return float64 holding the bf16 value.

    fp64 -> fp32 (RNE) -> bf16 (RNE); the GPU path rounds its fp32
    accumulator to bf16 the same way (C1.4)."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def rf32(x):
    """Round to fp32 (final logits / SSD heads stay fp32, C1.4)."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def bits_to_f64(b):
    return (np.ascontiguousarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def conv2d(x, w, b, stride=1, pad=0):
    """y[n,ho,wo,co] = b[co] + sum_{kh,kw,ci} xpad[n, ho*s+kh, wo*s+kw, ci] * w[co,kh,kw,ci].

    Zero padding, cross-correlation (C1.1); im2col + matmul per image."""
    N, H, W, C = x.shape
    Co, KH, KW, Ci = w.shape
    assert Ci == C, (Ci, C)
    Ho = (H + 2 * pad - KH) // stride + 1
    Wo = (W + 2 * pad - KW) // stride + 1
    wm = w.reshape(Co, KH * KW * C).T
    y = np.empty((N, Ho, Wo, Co), np.float64)
    for n in range(N):
        xp = np.zeros((H + 2 * pad, W + 2 * pad, C), np.float64)
        xp[pad:pad + H, pad:pad + W] = x[n]
        win = np.lib.stride_tricks.sliding_window_view(xp, (KH, KW), axis=(0, 1))
        # win: [H', W', C, KH, KW] -> select strided output positions
        win = win[: (Ho - 1) * stride + 1: stride, : (Wo - 1) * stride + 1: stride]
        cols = np.ascontiguousarray(win.transpose(0, 1, 3, 4, 2)).reshape(Ho * Wo, KH * KW * C)
        y[n] = (cols @ wm).reshape(Ho, Wo, Co)
    return y + b


def dwconv2d(x, w, b, stride=1, pad=1):
    """Depthwise conv (groups = C): y[n,ho,wo,c] = b[c] + sum_{kh,kw} xpad[..,c] * w[c,kh,kw,0]."""
    N, H, W, C = x.shape
    Cw, KH, KW, one = w.shape
    assert Cw == C and one == 1
    Ho = (H + 2 * pad - KH) // stride + 1
    Wo = (W + 2 * pad - KW) // stride + 1
    xp = np.zeros((N, H + 2 * pad, W + 2 * pad, C), np.float64)
    xp[:, pad:pad + H, pad:pad + W] = x
    y = np.zeros((N, Ho, Wo, C), np.float64)
    for kh in range(KH):
        for kw in range(KW):
            y += xp[:, kh: kh + (Ho - 1) * stride + 1: stride,
                    kw: kw + (Wo - 1) * stride + 1: stride, :] * w[:, kh, kw, 0]
    return y + b


def pool_out_size(H, k, s, pad, ceil):
    """PyTorch pooling output size; in ceil mode the last window must start
    inside the input or its left padding (C1.1)."""
    if ceil:
        o = -(-(H + 2 * pad - k) // s) + 1
        if (o - 1) * s >= H + pad:
            o -= 1
    else:
        o = (H + 2 * pad - k) // s + 1
    return o


def maxpool2d(x, k, s, pad=0, ceil=False):
    """Max over each k x k window (padding = -inf), NHWC."""
    N, H, W, C = x.shape
    Ho, Wo = pool_out_size(H, k, s, pad, ceil), pool_out_size(W, k, s, pad, ceil)
    Hp = max(H + 2 * pad, (Ho - 1) * s + k)
    Wp = max(W + 2 * pad, (Wo - 1) * s + k)
    xp = np.full((N, Hp, Wp, C), -np.inf)
    xp[:, pad:pad + H, pad:pad + W] = x
    y = np.full((N, Ho, Wo, C), -np.inf)
    for kh in range(k):
        for kw in range(k):
            y = np.maximum(y, xp[:, kh: kh + (Ho - 1) * s + 1: s, kw: kw + (Wo - 1) * s + 1: s, :])
    return y


def global_avgpool(x):
    """[N,H,W,C] -> [N,C] mean over H, W."""
    return x.mean(axis=(1, 2))


def linear(x, w, b):
    """y = x W^T + b, W [out, in]."""
    return x @ w.T + b


def relu(x):
    return np.maximum(x, 0.0)


def gelu(x):
    """GELU(erf): 0.5 x (1 + erf(x / sqrt 2))."""
    return 0.5 * x * (1.0 + erf(x / np.sqrt(2.0)))


def layernorm(x, g, b, eps=1e-12):
    """LN over the last axis, biased variance."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def softmax(x, axis=-1):
    """Max-subtracted softmax."""
    m = x.max(axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=axis, keepdims=True)
