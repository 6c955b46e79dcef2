"""Parameter manifests of the six models (names, shapes, init kinds) — data only.

Topologies are SURVEY.md §8(c) C1.2 readings of PAPER.md Table `tab:ml-models`
(names and input sizes only) plus the north_star's BERT-base (D1).
Shapes follow the layout convention of DESIGN.md §3:
  conv weight  [Cout, KH, KW, Cin]  (OHWI; depthwise: [C, 3, 3, 1])
  fc weight    [out, in]
  bias / LN    [C]
Init kinds (C1.3): "he" N(0, 2/fan_in); "he_q" = he * 0.25 (last conv of a
residual branch); "bias" U(-0.05, 0.05); "bert" N(0, 0.02^2); "ones"; "zeros".

Nothing here computes anything of the method; the oracle and the CUDA path
each walk their OWN topology and look parameters up by name.
"""

MODELS = ["lenet5", "googlenet", "resnet50", "ssd_mobilenet_v1", "vgg16", "bert_base"]
MODEL_INDEX = {m: i for i, m in enumerate(MODELS)}

# BERT-base reading: invented config.
BERT_LAYERS, BERT_H, BERT_HEADS, BERT_FFN, BERT_SEQ = 12, 768, 12, 3072, 128
BERT_VOCAB, BERT_MAXPOS, BERT_TYPES, BERT_CLASSES = 30522, 512, 2, 2

# GoogLeNet inception table: name, cin, c1, c3r, c3, c5r, c5, cpool
GOOGLENET_INCEPTION = [
    ("3a", 192, 64, 96, 128, 16, 32, 32),
    ("3b", 256, 128, 128, 192, 32, 96, 64),
    ("4a", 480, 192, 96, 208, 16, 48, 64),
    ("4b", 512, 160, 112, 224, 24, 64, 64),
    ("4c", 512, 128, 128, 256, 24, 64, 64),
    ("4d", 512, 112, 144, 288, 32, 64, 64),
    ("4e", 528, 256, 160, 320, 32, 128, 128),
    ("5a", 832, 256, 160, 320, 32, 128, 128),
    ("5b", 832, 384, 192, 384, 48, 128, 128),
]

# ResNet-50 stages: (blocks, width, first stride)
RESNET_STAGES = [(3, 64, 1), (4, 128, 2), (6, 256, 2), (3, 512, 2)]

# VGG-16 config D
VGG_CFG = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M",
           512, 512, 512, "M"]

# SSD-MobileNet-V1: MobileNet dw-separable blocks (cout, stride)
MOBILENET_BLOCKS = [(64, 1), (128, 2), (128, 1), (256, 2), (256, 1), (512, 2),
                    (512, 1), (512, 1), (512, 1), (512, 1), (512, 1), (1024, 2),
                    (1024, 1)]
SSD_EXTRAS = [(256, 512), (128, 256), (128, 256), (64, 128)]  # (1x1 mid, 3x3/2 out)
SSD_PRIORS, SSD_CLASSES = 6, 21


def _conv(out, name, cout, k, cin, init="he"):
    out.append((name + ".w", (cout, k, k, cin), init))
    out.append((name + ".b", (cout,), "bias"))


def _fc(out, name, nout, nin, init="he"):
    out.append((name + ".w", (nout, nin), init))
    out.append((name + ".b", (nout,), "bias"))


def _lenet():
    p = []
    _conv(p, "conv1", 6, 5, 1)
    _conv(p, "conv2", 16, 5, 6)
    _fc(p, "fc1", 120, 400)
    _fc(p, "fc2", 84, 120)
    _fc(p, "fc3", 10, 84)
    return p


def _resnet():
    p = []
    _conv(p, "conv1", 64, 7, 3)
    cin = 64
    for s, (nb, w, _stride) in enumerate(RESNET_STAGES):
        for i in range(nb):
            pre = f"layer{s + 1}.{i}"
            _conv(p, pre + ".conv1", w, 1, cin)
            _conv(p, pre + ".conv2", w, 3, w)
            _conv(p, pre + ".conv3", 4 * w, 1, w, init="he_q")
            if i == 0:
                _conv(p, pre + ".down", 4 * w, 1, cin)
            cin = 4 * w
    _fc(p, "fc", 1000, 2048)
    return p


def _vgg():
    p = []
    cin, n = 3, 0
    for v in VGG_CFG:
        if v == "M":
            continue
        n += 1
        _conv(p, f"conv{n}", v, 3, cin)
        cin = v
    _fc(p, "fc6", 4096, 7 * 7 * 512)
    _fc(p, "fc7", 4096, 4096)
    _fc(p, "fc8", 1000, 4096)
    return p


def _googlenet():
    p = []
    _conv(p, "conv1", 64, 7, 3)
    _conv(p, "conv2", 64, 1, 64)
    _conv(p, "conv3", 192, 3, 64)
    for name, cin, c1, c3r, c3, c5r, c5, cp in GOOGLENET_INCEPTION:
        pre = "inc" + name
        _conv(p, pre + ".b1", c1, 1, cin)
        _conv(p, pre + ".b2r", c3r, 1, cin)
        _conv(p, pre + ".b2", c3, 3, c3r)
        _conv(p, pre + ".b3r", c5r, 1, cin)
        _conv(p, pre + ".b3", c5, 5, c5r)
        _conv(p, pre + ".b4", cp, 1, cin)
    _fc(p, "fc", 1000, 1024)
    return p


def _ssd():
    p = []
    _conv(p, "conv0", 32, 3, 3)
    cin = 32
    for i, (cout, _s) in enumerate(MOBILENET_BLOCKS):
        p.append((f"dw{i + 1}.w", (cin, 3, 3, 1), "he"))
        p.append((f"dw{i + 1}.b", (cin,), "bias"))
        _conv(p, f"pw{i + 1}", cout, 1, cin)
        cin = cout
    for i, (mid, out) in enumerate(SSD_EXTRAS):
        _conv(p, f"extra{i + 1}.a", mid, 1, cin)
        _conv(p, f"extra{i + 1}.b", out, 3, mid)
        cin = out
    head_cin = [512, 1024] + [o for _m, o in SSD_EXTRAS]
    for i, c in enumerate(head_cin):
        _conv(p, f"head{i}.loc", SSD_PRIORS * 4, 3, c)
        _conv(p, f"head{i}.conf", SSD_PRIORS * SSD_CLASSES, 3, c)
    return p


def _bert():
    H, F = BERT_H, BERT_FFN
    p = [("emb.word", (BERT_VOCAB, H), "bert"), ("emb.pos", (BERT_MAXPOS, H), "bert"),
         ("emb.type", (BERT_TYPES, H), "bert"), ("emb.ln.g", (H,), "ones"),
         ("emb.ln.b", (H,), "zeros")]
    for i in range(BERT_LAYERS):
        pre = f"L{i}"
        _fc(p, pre + ".qkv", 3 * H, H, init="bert")
        _fc(p, pre + ".proj", H, H, init="bert")
        p += [(pre + ".ln1.g", (H,), "ones"), (pre + ".ln1.b", (H,), "zeros")]
        _fc(p, pre + ".ffn1", F, H, init="bert")
        _fc(p, pre + ".ffn2", H, F, init="bert")
        p += [(pre + ".ln2.g", (H,), "ones"), (pre + ".ln2.b", (H,), "zeros")]
    _fc(p, "pool", H, H, init="bert")
    _fc(p, "cls", BERT_CLASSES, H, init="bert")
    return p


_BUILDERS = {"lenet5": _lenet, "googlenet": _googlenet, "resnet50": _resnet,
             "ssd_mobilenet_v1": _ssd, "vgg16": _vgg, "bert_base": _bert}


def manifest(model):
    """[(name, shape, init_kind)] in file order for `model`."""
    return _BUILDERS[model]()


def input_shape(model, batch):
    """Logical input tensor shape (before the GPU's C 3->8 padding)."""
    return {"lenet5": (batch, 28, 28, 1), "googlenet": (batch, 224, 224, 3),
            "resnet50": (batch, 224, 224, 3), "vgg16": (batch, 224, 224, 3),
            "ssd_mobilenet_v1": (batch, 300, 300, 3),
            "bert_base": (batch, BERT_SEQ)}[model]
