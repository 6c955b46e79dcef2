"""Kernel parity on a B200: each layer kernel (through the C-ABI unit entry
points, run by the executor) vs the oracle's definition (oracle/nn.py) on the
same seeded bf16 inputs.  Shapes span several tiles and ragged tails."""
import numpy as np
import pytest

from oracle import nn
from tests.gpu_util import REL_TOL, bits_to_f64, from_dev_bf16, rel_err, to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2109_01611_b200 import gpulet
    c = gpulet.Context(1)
    yield c
    c.close()


def _bf16(rng, shape, scale=1.0):
    x = (rng.standard_normal(shape) * scale).astype(np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


GEMM_CASES = [(128, 64, 64, 1), (200, 96, 320, 1), (1000, 256, 768, 0), (77, 48, 1152, 2), (4096, 768, 3072, 0),
              (300, 1000, 512, 3), (513, 2304, 768, 0)]


@pytest.mark.parametrize("in_ws", [0, 1])
@pytest.mark.parametrize("M,N,K,act", GEMM_CASES)
def test_gemm_vs_oracle(ctx, M, N, K, act, in_ws):
    """in_ws=0: activation operand gathered by cp.async; in_ws=1: 2-D TMA."""
    import torch
    r = np.random.default_rng(M + N + K)
    A = _bf16(r, (M, K))
    W = _bf16(r, (N, K), 1 / np.sqrt(K))
    b = _bf16(r, (N,), 0.1)
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    ctx.test_gemm(0, to_dev_bf16(A), W, b, out, M, N, K, act=act, in_ws=in_ws)
    torch.cuda.synchronize()
    y = nn.linear(bits_to_f64(A), bits_to_f64(W), bits_to_f64(b))
    y = {0: y, 1: nn.relu(y), 2: nn.gelu(y), 3: np.tanh(y)}[act]
    ref = nn.rbf16(y)
    got = bits_to_f64(from_dev_bf16(out))
    assert rel_err(got, ref) < 1e-2
    # almost every element is bit-identical (differences are fp32 summation order only)
    assert np.mean(got == ref) > 0.9


# Paired ring stages (executor.cu gemm_step: two K blocks per stage on TMA-only steps
# while the ring keeps >= 3 stages, i.e. N tiles <= 128): odd K-block counts end in a
# one-block tail stage; N = 256 tiles keep one block per stage; forced split-K ranges
# (TUNE_SPLIT) have odd lengths and start at odd block offsets.
@pytest.mark.parametrize("splitk", [1, 3])
@pytest.mark.parametrize("M,N,K", [(300, 64, 64), (300, 64, 192), (260, 128, 320), (129, 96, 64 * 9),
                                   # >= 74 M blocks: the tile rule keeps N = 128 / 256 wide tiles
                                   (9500, 128, 320), (9500, 128, 448), (9500, 256, 192), (9500, 256, 320)])
def test_gemm_paired_stages_vs_oracle(ctx, M, N, K, splitk):
    import torch
    if splitk > K // 64:
        pytest.skip("fewer K blocks than splits")
    r = np.random.default_rng(M * 3 + N + K + splitk)
    A = _bf16(r, (M, K))
    W = _bf16(r, (N, K), 1 / np.sqrt(K))
    b = _bf16(r, (N,), 0.1)
    out = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    from paper_2109_01611_b200 import gpulet
    gpulet.Context.set_tuning(1, splitk if splitk > 1 else 0)   # TUNE_SPLIT: force the split count
    try:
        ctx.test_gemm(0, to_dev_bf16(A), W, b, out, M, N, K, act=1, splitk=1, in_ws=1)
    finally:
        gpulet.Context.set_tuning(1, 0)
    torch.cuda.synchronize()
    ref = nn.rbf16(nn.relu(nn.linear(bits_to_f64(A), bits_to_f64(W), bits_to_f64(b))))
    got = bits_to_f64(from_dev_bf16(out))
    assert rel_err(got, ref) < 1e-2
    assert np.mean(got == ref) > 0.9


@pytest.mark.parametrize("in_ws", [0, 1])
@pytest.mark.parametrize("M,N,K", [(1, 1000, 2048), (7, 4096, 25088), (32, 1000, 4096), (16, 2, 768), (3, 768, 768)])
def test_gemm_swap_ab_splitk_vs_oracle(ctx, M, N, K, in_ws):
    import torch
    r = np.random.default_rng(M * 7 + N)
    A = _bf16(r, (M, K))
    W = _bf16(r, (N, K), 1 / np.sqrt(K))
    b = _bf16(r, (N,), 0.1)
    out = torch.empty((M, N), dtype=torch.float32, device="cuda")
    ctx.test_gemm(0, to_dev_bf16(A), W, b, out, M, N, K, act=0, swap_ab=1, out_fp32=1, in_ws=in_ws)
    torch.cuda.synchronize()
    ref = nn.linear(bits_to_f64(A), bits_to_f64(W), bits_to_f64(b))
    assert rel_err(out.cpu().numpy(), ref) < 1e-4


CONV_CASES = [(2, 14, 14, 64, 128, 3, 1, 1), (1, 30, 30, 8, 64, 7, 2, 3), (2, 9, 9, 32, 24, 3, 2, 1),
              (3, 15, 15, 256, 512, 1, 2, 0), (1, 12, 12, 16, 48, 5, 1, 2), (2, 19, 19, 512, 126, 3, 1, 1),
              (1, 56, 56, 64, 64, 3, 1, 1), (2, 28, 28, 128, 128, 3, 2, 1), (2, 10, 10, 256, 512, 3, 2, 1),
              (3, 7, 7, 512, 256, 1, 1, 0), (2, 5, 5, 128, 64, 5, 1, 2), (2, 14, 14, 96, 128, 3, 1, 1),
              (1, 14, 14, 24, 64, 5, 1, 2), (2, 7, 7, 160, 320, 3, 1, 1), (2, 28, 28, 48, 128, 5, 1, 2),
              (4, 32, 32, 8, 64, 3, 1, 1), (2, 32, 32, 8, 64, 7, 2, 3), (2, 30, 30, 8, 32, 3, 2, 1)]


@pytest.mark.parametrize("in_ws", [0, 1, 2])
@pytest.mark.parametrize("N,H,W,C,Co,k,s,p", CONV_CASES)
def test_conv_vs_oracle(ctx, N, H, W, C, Co, k, s, p, in_ws):
    """in_ws=0: cp.async implicit-im2col gather (forced by tuning key 4);
    in_ws=1: TMA (2-D for 1x1/s1, im2col boxes of 64/32/16/8 channels otherwise);
    in_ws=2: input at the request address, staged into the workspace by the
    program (copy, 2x2 space-to-depth or kw-packing for small-C convs)."""
    import torch
    from paper_2109_01611_b200 import gpulet
    r = np.random.default_rng(H * C + Co)
    x = _bf16(r, (N, H, W, C))
    w = _bf16(r, (Co, k, k, C), np.sqrt(2 / (k * k * C)))
    b = _bf16(r, (Co,), 0.05)
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    y = torch.empty((N, Ho, Wo, Co), dtype=torch.bfloat16, device="cuda")
    gpulet.Context.set_tuning(4, 1 if in_ws == 0 else 0)
    try:
        ctx.test_conv(0, to_dev_bf16(x), w, b, y, N, H, W, C, Co, k, s, p, act=1, in_ws=1 if in_ws == 1 else 0)
    finally:
        gpulet.Context.set_tuning(4, 0)
    torch.cuda.synchronize()
    ref = nn.rbf16(nn.relu(nn.conv2d(bits_to_f64(x), bits_to_f64(w), bits_to_f64(b), s, p)))
    got = bits_to_f64(from_dev_bf16(y))
    assert rel_err(got, ref) < 1e-2
    assert np.mean(got == ref) > 0.9


@pytest.mark.parametrize("s", [1, 2])
def test_dwconv_vs_oracle(ctx, s):
    import torch
    r = np.random.default_rng(s)
    N, H, W, C = 2, 19, 19, 64
    x = _bf16(r, (N, H, W, C))
    w = _bf16(r, (C, 3, 3, 1), 0.5)
    b = _bf16(r, (C,), 0.05)
    Ho = (H + 2 - 3) // s + 1
    y = torch.empty((N, Ho, Ho, C), dtype=torch.bfloat16, device="cuda")
    ctx.test_misc(0, 2, [N, H, W, C, s], np.concatenate([w.reshape(-1), b]), to_dev_bf16(x), y)
    torch.cuda.synchronize()
    ref = nn.rbf16(nn.relu(nn.dwconv2d(bits_to_f64(x), bits_to_f64(w), bits_to_f64(b), s, 1)))
    assert rel_err(bits_to_f64(from_dev_bf16(y)), ref) < 1e-2


@pytest.mark.parametrize("k,s,p,ceil,H", [(3, 2, 1, False, 112), (3, 2, 0, True, 112), (3, 2, 0, True, 14),
                                           (2, 2, 0, False, 28), (3, 1, 1, False, 7)])
def test_maxpool_bit_exact(ctx, k, s, p, ceil, H):
    import torch
    r = np.random.default_rng(H + k)
    x = _bf16(r, (2, H, H, 16))
    Ho = nn.pool_out_size(H, k, s, p, ceil)
    y = torch.empty((2, Ho, Ho, 16), dtype=torch.bfloat16, device="cuda")
    ctx.test_misc(0, 3, [2, H, H, 16, k, s, p, int(ceil)], None, to_dev_bf16(x), y)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(bits_to_f64(from_dev_bf16(y)), nn.maxpool2d(bits_to_f64(x), k, s, p, ceil))


def test_avgpool(ctx):
    import torch
    r = np.random.default_rng(9)
    x = _bf16(r, (3, 7, 7, 2048))
    y = torch.empty((3, 2048), dtype=torch.bfloat16, device="cuda")
    ctx.test_misc(0, 4, [3, 7, 7, 2048], None, to_dev_bf16(x), y)
    torch.cuda.synchronize()
    ref = nn.rbf16(nn.global_avgpool(bits_to_f64(x)))
    assert rel_err(bits_to_f64(from_dev_bf16(y)), ref) < 1e-2


def test_layernorm(ctx):
    import torch
    r = np.random.default_rng(10)
    x = _bf16(r, (300, 768), 2.0)
    g = _bf16(r, (768,))
    b = _bf16(r, (768,))
    y = torch.empty((300, 768), dtype=torch.bfloat16, device="cuda")
    ctx.test_misc(0, 7, [300], np.concatenate([g, b]), to_dev_bf16(x), y)
    torch.cuda.synchronize()
    ref = nn.rbf16(nn.layernorm(bits_to_f64(x), bits_to_f64(g), bits_to_f64(b)))
    assert rel_err(bits_to_f64(from_dev_bf16(y)), ref) < 1e-2


@pytest.mark.parametrize("tensor_core", [1, 0])
def test_attention(ctx, tensor_core):
    import torch
    r = np.random.default_rng(11)
    nseq = 3
    qkv = _bf16(r, (nseq * 128, 3 * 768))
    y = torch.empty((nseq * 128, 768), dtype=torch.bfloat16, device="cuda")
    ctx.test_misc(0, 8, [nseq, tensor_core], None, to_dev_bf16(qkv), y)
    torch.cuda.synchronize()
    q = bits_to_f64(qkv).reshape(nseq, 128, 3, 12, 64)
    s = np.einsum("bqhd,bkhd->bhqk", q[:, :, 0], q[:, :, 1]) * 0.125
    p = nn.rbf16(nn.softmax(s, -1))
    ref = nn.rbf16(np.einsum("bhqk,bkhd->bqhd", p, q[:, :, 2])).reshape(nseq * 128, 768)
    assert rel_err(bits_to_f64(from_dev_bf16(y)), ref) < 2e-2


def test_softmax(ctx):
    import torch
    r = np.random.default_rng(12)
    x = (r.standard_normal((1000, 21)) * 3).astype(np.float32)
    t = torch.from_numpy(x).cuda()
    ctx.test_misc(0, 9, [1000, 21], None, None, t)
    torch.cuda.synchronize()
    np.testing.assert_allclose(t.cpu().numpy(), nn.softmax(x.astype(np.float64)), rtol=1e-5, atol=1e-7)
