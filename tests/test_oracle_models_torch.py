"""Whole-model pins of the C1 forward-pass oracle (oracle/models.py) against
independent torch-CPU fp64 references built from the standard layouts — the
wiring the layer pins cannot see (VERDICT r1 "What's weak" 2): residual add
before ReLU and v1.5 strides (torchvision resnet50), the NHWC flatten before
the first FC (torchvision vgg16 / the LeNet-5 layout with fc columns permuted),
Inception branch order and true 5x5 branch (torchvision GoogLeNet blocks with
the 5x5 conv restored and 3x3/2 ceil pools), BERT's (S, 3, NH, DH)
QKV split and post-LN placement (nn.TransformerEncoderLayer norm_first=False,
activation gelu), SSD's (h, w, prior) head order (permute + reshape, the
torchvision SSD convention).

With the C1.4 bf16 rounding switched off (pure fp64 on both sides) the
oracle must agree with the reference to 1e-9 relative.  Weights and inputs are
the seeded synthetic ones (synthgen); BN layers of the torchvision modules are
set to an exact affine "+ bias" (running var 1 - eps, mean 0, gamma 1)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthgen
from oracle import models as om
from oracle import nn as onn

pytestmark = pytest.mark.slow
TOL = 1e-9


@pytest.fixture
def no_rounding(monkeypatch):
    ident = lambda x: np.asarray(x, dtype=np.float64)  # noqa: E731
    monkeypatch.setattr(om, "R", ident)
    monkeypatch.setattr(onn, "rf32", ident)


def _w(wb, name):
    return torch.from_numpy(onn.bits_to_f64(wb[name]))


def _conv_w(wb, name):
    return _w(wb, name + ".w").permute(0, 3, 1, 2).contiguous()     # OHWI -> OIHW


def _x(model, b):
    x = synthgen.model_input(model, b)
    return x, torch.from_numpy(onn.bits_to_f64(x)).permute(0, 3, 1, 2).contiguous()


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b).max() / np.abs(b).max()


def _bias_bn(bn, bias):
    """BatchNorm2d (eval) reduced to + bias."""
    bn.eval()
    with torch.no_grad():
        bn.weight.fill_(1.0)
        bn.bias.copy_(bias)
        bn.running_mean.zero_()
        bn.running_var.fill_(1.0 - bn.eps)


def _set_conv(conv, bn, wb, name):
    with torch.no_grad():
        conv.weight.copy_(_conv_w(wb, name))
    _bias_bn(bn, _w(wb, name + ".b"))


def test_resnet50_equals_torchvision(no_rounding):
    import torchvision
    wb = synthgen.weights("resnet50")
    net = torchvision.models.resnet50(weights=None).double().eval()
    _set_conv(net.conv1, net.bn1, wb, "conv1")
    for s in range(4):
        for i, blk in enumerate(getattr(net, f"layer{s + 1}")):
            pre = f"layer{s + 1}.{i}"
            _set_conv(blk.conv1, blk.bn1, wb, pre + ".conv1")
            _set_conv(blk.conv2, blk.bn2, wb, pre + ".conv2")
            _set_conv(blk.conv3, blk.bn3, wb, pre + ".conv3")
            if blk.downsample is not None:
                _set_conv(blk.downsample[0], blk.downsample[1], wb, pre + ".down")
    with torch.no_grad():
        net.fc.weight.copy_(_w(wb, "fc.w"))
        net.fc.bias.copy_(_w(wb, "fc.b"))
    x, xt = _x("resnet50", 2)
    with torch.no_grad():
        ref = net(xt).numpy()
    got = om.forward("resnet50", wb, x)["logits"]
    assert _rel(got, ref) <= TOL


def _fc_nhwc_to_nchw(w, C, H, W):
    """fc weight over an NHWC flatten (h, w, c) -> the same map over an NCHW flatten (c, h, w)."""
    return w.reshape(w.shape[0], H, W, C).permute(0, 3, 1, 2).reshape(w.shape[0], -1)


def test_vgg16_equals_torchvision(no_rounding):
    import torchvision
    wb = synthgen.weights("vgg16")
    net = torchvision.models.vgg16(weights=None).double().eval()
    convs = [m for m in net.features if isinstance(m, torch.nn.Conv2d)]
    assert len(convs) == 13
    with torch.no_grad():
        for n, c in enumerate(convs):
            c.weight.copy_(_conv_w(wb, f"conv{n + 1}"))
            c.bias.copy_(_w(wb, f"conv{n + 1}.b"))
        fcs = [m for m in net.classifier if isinstance(m, torch.nn.Linear)]
        fcs[0].weight.copy_(_fc_nhwc_to_nchw(_w(wb, "fc6.w"), 512, 7, 7))
        fcs[0].bias.copy_(_w(wb, "fc6.b"))
        for m, name in zip(fcs[1:], ("fc7", "fc8")):
            m.weight.copy_(_w(wb, name + ".w"))
            m.bias.copy_(_w(wb, name + ".b"))
    x, xt = _x("vgg16", 1)
    with torch.no_grad():
        ref = net(xt).numpy()
    got = om.forward("vgg16", wb, x)["logits"]
    assert _rel(got, ref) <= TOL


def test_lenet5_equals_functional(no_rounding):
    wb = synthgen.weights("lenet5")
    x, xt = _x("lenet5", 4)
    h = F.max_pool2d(F.relu(F.conv2d(xt, _conv_w(wb, "conv1"), _w(wb, "conv1.b"), padding=2)), 2)
    h = F.max_pool2d(F.relu(F.conv2d(h, _conv_w(wb, "conv2"), _w(wb, "conv2.b"))), 2)
    h = h.flatten(1)                                                 # NCHW flatten
    h = F.relu(F.linear(h, _fc_nhwc_to_nchw(_w(wb, "fc1.w"), 16, 5, 5), _w(wb, "fc1.b")))
    h = F.relu(F.linear(h, _w(wb, "fc2.w"), _w(wb, "fc2.b")))
    ref = F.linear(h, _w(wb, "fc3.w"), _w(wb, "fc3.b")).numpy()
    assert _rel(om.forward("lenet5", wb, x)["logits"], ref) <= TOL


def test_googlenet_equals_torchvision_blocks(no_rounding):
    """torchvision's GoogLeNet module graph (stem, Inception blocks: branch order
    1x1 | 1x1->3x3 | 1x1->5x5 | pool->1x1, concat on channels), with its two
    known deviations from Inception-v1 undone: the 5x5 branch (torchvision: 3x3)
    and the 3x3/2 pool before 5a (torchvision: 2x2)."""
    import torchvision
    from torchvision.models.googlenet import BasicConv2d
    wb = synthgen.weights("googlenet")
    net = torchvision.models.GoogLeNet(num_classes=1000, aux_logits=False, transform_input=False,
                                       init_weights=False).double().eval()
    net.maxpool4 = torch.nn.MaxPool2d(3, 2, ceil_mode=True)

    def setb(bc, name):
        _set_conv(bc.conv, bc.bn, wb, name)
    setb(net.conv1, "conv1")
    setb(net.conv2, "conv2")
    setb(net.conv3, "conv3")
    for name in ("3a", "3b", "4a", "4b", "4c", "4d", "4e", "5a", "5b"):
        blk = getattr(net, "inception" + name)
        pre = "inc" + name
        w5 = wb[pre + ".b3.w"]
        blk.branch3[1] = BasicConv2d(w5.shape[3], w5.shape[0], kernel_size=5, padding=2).double().eval()
        setb(blk.branch1, pre + ".b1")
        setb(blk.branch2[0], pre + ".b2r")
        setb(blk.branch2[1], pre + ".b2")
        setb(blk.branch3[0], pre + ".b3r")
        setb(blk.branch3[1], pre + ".b3")
        setb(blk.branch4[1], pre + ".b4")
    with torch.no_grad():
        net.fc.weight.copy_(_w(wb, "fc.w"))
        net.fc.bias.copy_(_w(wb, "fc.b"))
    x, xt = _x("googlenet", 1)
    with torch.no_grad():
        ref = net(xt).numpy()
    assert _rel(om.forward("googlenet", wb, x)["logits"], ref) <= TOL


def test_ssd_mobilenet_equals_functional(no_rounding):
    """MobileNet-V1 (3x3/2 stem, 13 depthwise-separable blocks), 4 extras (1x1 then
    3x3/2), 3x3 heads on the 19/10/5/3/2/1 maps; head outputs permuted NCHW -> NHWC and
    reshaped to (h, w, prior) rows; softmax over the 21 classes."""
    wb = synthgen.weights("ssd_mobilenet_v1")
    blocks = [(64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2), (512, 1), (512, 1), (512, 1), (512, 1),
              (512, 1), (1024, 2), (1024, 1)]
    x, h = _x("ssd_mobilenet_v1", 1)

    def conv(h, name, stride=1, pad=0, groups=1):
        return F.conv2d(h, _conv_w(wb, name), _w(wb, name + ".b"), stride=stride, padding=pad, groups=groups)
    h = F.relu(conv(h, "conv0", 2, 1))
    feats = []
    for i, (_c, s) in enumerate(blocks):
        h = F.relu(conv(h, f"dw{i + 1}", s, 1, groups=h.shape[1]))
        h = F.relu(conv(h, f"pw{i + 1}"))
        if i + 1 in (11, 13):
            feats.append(h)
    for i in range(4):
        h = F.relu(conv(h, f"extra{i + 1}.a"))
        h = F.relu(conv(h, f"extra{i + 1}.b", 2, 1))
        feats.append(h)
    assert [f.shape[-1] for f in feats] == [19, 10, 5, 3, 2, 1]
    loc = torch.cat([conv(f, f"head{i}.loc", 1, 1).permute(0, 2, 3, 1).reshape(1, -1, 4)
                     for i, f in enumerate(feats)], 1)
    conf = torch.cat([conv(f, f"head{i}.conf", 1, 1).permute(0, 2, 3, 1).reshape(1, -1, 21)
                      for i, f in enumerate(feats)], 1).softmax(-1)
    got = om.forward("ssd_mobilenet_v1", wb, x)
    assert loc.shape[1] == 3000
    assert _rel(got["loc"], loc.numpy()) <= TOL
    assert _rel(got["conf"], conf.numpy()) <= TOL


def test_bert_equals_transformer_encoder(no_rounding):
    wb = synthgen.weights("bert_base")
    ids = synthgen.model_input("bert_base", 2)
    W = lambda n: _w(wb, n)  # noqa: E731
    it = torch.from_numpy(ids).long()
    e = W("emb.word")[it] + W("emb.pos")[: ids.shape[1]][None] + W("emb.type")[0][None, None]
    h = F.layer_norm(e, (768,), W("emb.ln.g"), W("emb.ln.b"), eps=1e-12)
    for i in range(12):
        p = f"L{i}."
        layer = torch.nn.TransformerEncoderLayer(768, 12, 3072, dropout=0.0, activation="gelu", batch_first=True,
                                                 norm_first=False, layer_norm_eps=1e-12).double().eval()
        with torch.no_grad():
            layer.self_attn.in_proj_weight.copy_(W(p + "qkv.w"))
            layer.self_attn.in_proj_bias.copy_(W(p + "qkv.b"))
            layer.self_attn.out_proj.weight.copy_(W(p + "proj.w"))
            layer.self_attn.out_proj.bias.copy_(W(p + "proj.b"))
            layer.linear1.weight.copy_(W(p + "ffn1.w"))
            layer.linear1.bias.copy_(W(p + "ffn1.b"))
            layer.linear2.weight.copy_(W(p + "ffn2.w"))
            layer.linear2.bias.copy_(W(p + "ffn2.b"))
            layer.norm1.weight.copy_(W(p + "ln1.g"))
            layer.norm1.bias.copy_(W(p + "ln1.b"))
            layer.norm2.weight.copy_(W(p + "ln2.g"))
            layer.norm2.bias.copy_(W(p + "ln2.b"))
            h = layer(h)
    with torch.no_grad():
        pooled = torch.tanh(F.linear(h[:, 0], W("pool.w"), W("pool.b")))
        ref = F.linear(pooled, W("cls.w"), W("cls.b")).numpy()
    assert _rel(om.forward("bert_base", wb, ids)["logits"], ref) <= TOL
