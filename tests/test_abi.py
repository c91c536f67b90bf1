"""The C-ABI boundary: both shared libraries load without a GPU and export every
function the headers in include/ declare; on a machine without a B200 the GPU
library refuses to create a context (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2403_02310_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_][a-z0-9_]*\s*\**\s+\**\s*(ss[h]?_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.mark.parametrize("header,loader", [("ss_gpu.h", _lib.gpu_lib), ("ss_host.h", _lib.host_lib)])
def test_exports_every_declared_symbol(header, loader):
    lib = loader()
    names = declared(header)
    assert len(names) > 10, names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_lists_match_headers():
    assert set(_lib.GPU_EXPORTS) == set(declared("ss_gpu.h"))
    assert set(_lib.HOST_EXPORTS) == set(declared("ss_host.h"))


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2403_02310_b200 import gpu

    with pytest.raises(_lib.SSError) as ei:
        gpu.HybridForward(gpu.MODELS["tiny"])
    assert "no CUDA device" in str(ei.value)


def test_kernel_class_names():
    lib = _lib.gpu_lib()
    from paper_2403_02310_b200.gpu import KERNEL_CLASSES

    assert [lib.ss_kernel_class_name(i).decode() for i in range(len(KERNEL_CLASSES))] == KERNEL_CLASSES
