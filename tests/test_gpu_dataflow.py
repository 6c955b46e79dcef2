"""Barrier-free GEMM step joins (gl_set_tuning(6, 1), off by default):
the same parity bar with the gpu-let barrier replaced by per-M-block
completion counters between consecutive TMA GEMM steps.  Runs in a child
process because the switch applies to programs built afterwards."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import numpy as np, torch, synthgen
from oracle import models as om
from paper_2109_01611_b200 import gpulet
from tools import common
from tests.gpu_util import rel_err, REL_TOL
gpulet.Context.set_tuning(6, 2)   # dataflow joins + plan log
ctx = gpulet.Context(1)
for m, b in (("resnet50", 3), ("vgg16", 2)):
    mid = ctx.load_model(0, m, synthgen.weight_file(m))
    x = common.device_input(m, b)
    y = torch.empty(ctx.model_io(mid, b)[1] // 4, device="cuda")
    for _ in range(2):   # the second run checks the counters were re-zeroed
        ctx.run_once(mid, b, x, y, 0, True)
        got = y.cpu().numpy().astype(np.float64).reshape(b, -1)
        ref = om.forward(m, synthgen.weights(m), synthgen.model_input(m, b))["logits"].reshape(b, -1)
        e = rel_err(got, ref)
        assert e <= REL_TOL, (m, e)
    print(m, "ok", e)
ctx.close()
'''


def test_dataflow_joins_parity():
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "barrier-free joins" in r.stderr          # the joins were planned
    assert "resnet50 ok" in r.stdout and "vgg16 ok" in r.stdout
