"""The C-ABI library builds, loads without a GPU and exports every function
include/gpulet.h declares; host-only entry points behave (no compute calls)."""
import ctypes
import os
import re

import pytest

from paper_2109_01611_b200 import gpulet

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "gpulet.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gl_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(gpulet.LIB_PATH):
        from paper_2109_01611_b200 import build
        build.build(verbose=False)
    return gpulet.lib()


def test_exports_every_declared_symbol(lib):
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(gpulet.SYMBOLS) == names


def test_no_torch_in_abi():
    src = open(HDR).read()
    code = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    assert "torch" not in code and "std::" not in code and "class " not in code
    assert 'extern "C"' in src


def test_host_only_calls_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only checks")
    h = ctypes.c_void_p()
    assert lib.gl_init(1, ctypes.byref(h)) == -12          # GL_E_CUDA: no device, fails loudly
    assert lib.gl_last_error()
    assert lib.gl_init(0, ctypes.byref(h)) == -1           # GL_E_ARG
    assert lib.gl_shutdown(None) == 0


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", gpulet.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", gpulet.LIB_PATH], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):          # tcgen05.mma, TMA, tcgen05.ld
        assert mnemonic in sass, mnemonic
