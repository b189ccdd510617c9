"""Every C entry point declared in include/*.h is exported by the in-tree
libraries (loads without a GPU)."""
import ctypes
import os
import re

from paper_1901_06773_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(accudnn_\w+)\s*\(", text)))


def test_planner_abi_exports():
    lib = _native.planner_lib()
    names = declared("accudnn_plan.h")
    assert len(names) >= 10
    for n in names:
        assert hasattr(lib, n), n


def test_runtime_and_kernel_abi_exports():
    lib = _native.cuda_lib()
    for h in ("accudnn.h", "accudnn_kernels.h"):
        names = declared(h)
        assert len(names) >= 10
        for n in names:
            assert hasattr(lib, n), (h, n)


def test_no_cpu_fallback_symbols():
    """The product path has no host implementation of the layer math: the
    kernel library exports launchers only (no *_cpu / *_reference entry)."""
    lib = _native.cuda_lib()
    for suffix in ("cpu", "reference", "fallback"):
        assert not hasattr(lib, f"accudnn_conv_fwd_{suffix}")
