"""C1.2 model forward passes (ORACLE — test infrastructure only).

Topologies: SURVEY.md §8(c) C1.2 readings (the paper names the models and
their input sizes only, Table `tab:ml-models`; BERT-base is a
north_star addition, D1).  Quantisation points: C1.4 — every layer consumes
bf16 values, accumulates exactly (fp64 here), and its epilogue applies
+bias -> (+bf16 residual) -> activation -> round-to-bf16.  Final logits and the
SSD heads stay fp32.  Parity status: pinned.  The layer maths against torch-CPU
and brute force (test_oracle_nn); the closed-form MAC / parameter totals
(test_oracle_models); and each whole model, with the bf16 rounding switched off,
against an independent torch-CPU fp64 reference in its standard layout to 1e-9
(test_oracle_models_torch: torchvision resnet50 / vgg16 / GoogLeNet blocks,
nn.TransformerEncoderLayer for BERT, torch.nn.functional LeNet-5 and SSD), which
fixes the wiring the totals cannot see (residual order, flatten order, branch
order, QKV split, post-LN placement, head order).  The topologies remain
readings of the paper (C6 #1-#4: it names the models and input sizes only).
"""
import numpy as np

from . import nn

R = nn.rbf16


class _W:
    """Parameter accessor (bf16 bits -> float64), records MACs for pins."""

    def __init__(self, wbits):
        self.w = wbits
        self.macs = 0

    def __getitem__(self, k):
        return nn.bits_to_f64(self.w[k])

    def conv(self, x, name, stride=1, pad=0):
        w = self[name + ".w"]
        y = nn.conv2d(x, w, self[name + ".b"], stride, pad)
        self.macs += y.shape[0] * y.shape[1] * y.shape[2] * w.size
        return y

    def dw(self, x, name, stride):
        w = self[name + ".w"]
        y = nn.dwconv2d(x, w, self[name + ".b"], stride, 1)
        self.macs += y.shape[0] * y.shape[1] * y.shape[2] * w.size
        return y

    def fc(self, x, name):
        w = self[name + ".w"]
        self.macs += x.shape[0] * w.size
        return nn.linear(x, w, self[name + ".b"])


def lenet5(P, x):
    """LeNet-5 [b,28,28,1] -> logits [b,10] (fp32)."""
    h = R(nn.relu(P.conv(x, "conv1", 1, 2)))
    h = nn.maxpool2d(h, 2, 2)
    h = R(nn.relu(P.conv(h, "conv2", 1, 0)))
    h = nn.maxpool2d(h, 2, 2)
    h = h.reshape(h.shape[0], -1)                       # NHWC flatten (h, w, c)
    h = R(nn.relu(P.fc(h, "fc1")))
    h = R(nn.relu(P.fc(h, "fc2")))
    return {"logits": nn.rf32(P.fc(h, "fc3"))}


RESNET_STAGES = [(3, 64, 1), (4, 128, 2), (6, 256, 2), (3, 512, 2)]


def resnet50(P, x):
    """ResNet-50 v1.5 (stride on the 3x3), BN folded into conv bias."""
    h = R(nn.relu(P.conv(x, "conv1", 2, 3)))
    h = nn.maxpool2d(h, 3, 2, 1)
    for s, (nb, _w, stride) in enumerate(RESNET_STAGES):
        for i in range(nb):
            pre = f"layer{s + 1}.{i}"
            st = stride if i == 0 else 1
            a = R(nn.relu(P.conv(h, pre + ".conv1")))
            a = R(nn.relu(P.conv(a, pre + ".conv2", st, 1)))
            sc = R(P.conv(h, pre + ".down", st)) if i == 0 else h
            h = R(nn.relu(P.conv(a, pre + ".conv3") + sc))
    h = R(nn.global_avgpool(h))
    return {"logits": nn.rf32(P.fc(h, "fc"))}


VGG_CFG = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
           512, 512, 512, "M"]


def vgg16(P, x):
    """VGG-16 config D, no BN; NHWC flatten before fc6."""
    h, n = x, 0
    for v in VGG_CFG:
        if v == "M":
            h = nn.maxpool2d(h, 2, 2)
        else:
            n += 1
            h = R(nn.relu(P.conv(h, f"conv{n}", 1, 1)))
    h = h.reshape(h.shape[0], -1)
    h = R(nn.relu(P.fc(h, "fc6")))
    h = R(nn.relu(P.fc(h, "fc7")))
    return {"logits": nn.rf32(P.fc(h, "fc8"))}


GOOGLENET_INCEPTION = ["3a", "3b", "P", "4a", "4b", "4c", "4d", "4e", "P", "5a", "5b"]


def googlenet(P, x):
    """Inception-v1 without aux heads/LRN, true 5x5 branch, 3x3/2 ceil-mode pools."""
    h = R(nn.relu(P.conv(x, "conv1", 2, 3)))
    h = nn.maxpool2d(h, 3, 2, 0, ceil=True)
    h = R(nn.relu(P.conv(h, "conv2")))
    h = R(nn.relu(P.conv(h, "conv3", 1, 1)))
    h = nn.maxpool2d(h, 3, 2, 0, ceil=True)
    for name in GOOGLENET_INCEPTION:
        if name == "P":
            h = nn.maxpool2d(h, 3, 2, 0, ceil=True)
            continue
        pre = "inc" + name
        b1 = R(nn.relu(P.conv(h, pre + ".b1")))
        b2 = R(nn.relu(P.conv(R(nn.relu(P.conv(h, pre + ".b2r"))), pre + ".b2", 1, 1)))
        b3 = R(nn.relu(P.conv(R(nn.relu(P.conv(h, pre + ".b3r"))), pre + ".b3", 1, 2)))
        b4 = R(nn.relu(P.conv(nn.maxpool2d(h, 3, 1, 1), pre + ".b4")))
        h = np.concatenate([b1, b2, b3, b4], axis=-1)   # branch order 1x1, 3x3, 5x5, pool
    h = R(nn.global_avgpool(h))
    return {"logits": nn.rf32(P.fc(h, "fc"))}


MOBILENET_BLOCKS = [(64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2),
                    (512, 1), (512, 1), (512, 1), (512, 1), (512, 1), (1024, 2),
                    (1024, 1)]


def ssd_mobilenet_v1(P, x):
    """MobileNet-V1 + 4 SSD extras + 3x3 loc/conf heads on maps 19,10,5,3,2,1
    (6 priors each = 3000 priors, 21 classes); conf softmax in fp32."""
    h = R(nn.relu(P.conv(x, "conv0", 2, 1)))
    feats = []
    for i, (_c, s) in enumerate(MOBILENET_BLOCKS):
        h = R(nn.relu(P.dw(h, f"dw{i + 1}", s)))
        h = R(nn.relu(P.conv(h, f"pw{i + 1}")))
        if i + 1 in (11, 13):
            feats.append(h)
    for i in range(4):
        h = R(nn.relu(P.conv(h, f"extra{i + 1}.a")))
        h = R(nn.relu(P.conv(h, f"extra{i + 1}.b", 2, 1)))
        feats.append(h)
    locs, confs = [], []
    for i, f in enumerate(feats):
        lo = nn.rf32(P.conv(f, f"head{i}.loc", 1, 1))
        co = nn.rf32(P.conv(f, f"head{i}.conf", 1, 1))
        locs.append(lo.reshape(lo.shape[0], -1, 4))      # (h, w, prior) order
        confs.append(co.reshape(co.shape[0], -1, 21))
    loc = np.concatenate(locs, axis=1)
    conf = nn.rf32(nn.softmax(np.concatenate(confs, axis=1), axis=-1))
    return {"loc": loc, "conf": conf}


BERT_L, BERT_H, BERT_NH, BERT_DH = 12, 768, 12, 64


def bert_base(P, ids):
    """BERT-base encoder (seq 128, no mask) + pooler(tanh) + 2-class head."""
    b, S = ids.shape
    word, pos, typ = P["emb.word"], P["emb.pos"], P["emb.type"]
    e = word[ids] + pos[:S][None] + typ[0][None, None]
    x = R(nn.layernorm(e, P["emb.ln.g"], P["emb.ln.b"])).reshape(b * S, BERT_H)
    for i in range(BERT_L):
        pre = f"L{i}"
        qkv = R(P.fc(x, pre + ".qkv")).reshape(b, S, 3, BERT_NH, BERT_DH)
        q, k, v = qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]          # [b,S,NH,DH]
        s = np.einsum("bqhd,bkhd->bhqk", q, k) * 0.125
        p = R(nn.softmax(s, axis=-1))
        o = R(np.einsum("bhqk,bkhd->bqhd", p, v)).reshape(b * S, BERT_H)
        P.macs += 2 * b * BERT_NH * S * S * BERT_DH
        a = R(P.fc(o, pre + ".proj") + x)
        x = R(nn.layernorm(a, P[pre + ".ln1.g"], P[pre + ".ln1.b"]))
        f = R(nn.gelu(P.fc(x, pre + ".ffn1")))
        y = R(P.fc(f, pre + ".ffn2") + x)
        x = R(nn.layernorm(y, P[pre + ".ln2.g"], P[pre + ".ln2.b"]))
    cls = x.reshape(b, S, BERT_H)[:, 0]
    pooled = R(np.tanh(P.fc(cls, "pool")))
    return {"logits": nn.rf32(P.fc(pooled, "cls")), "pooled": pooled}


FORWARD = {"lenet5": lenet5, "googlenet": googlenet, "resnet50": resnet50,
           "ssd_mobilenet_v1": ssd_mobilenet_v1, "vgg16": vgg16, "bert_base": bert_base}


def forward(model, wbits, x, return_macs=False):
    """Run `model` on input `x` (bf16 bits NHWC for images, int32 ids for BERT).

    wbits: {name: uint16 bf16 bits} as drawn by synthgen."""
    P = _W(wbits)
    xin = x if model == "bert_base" else nn.bits_to_f64(x)
    out = FORWARD[model](P, xin)
    if return_macs:
        return out, P.macs // x.shape[0]   # MACs per request
    return out
