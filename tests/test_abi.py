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


def test_committed_conv_tune_table_round_trips():
    """profiles/b200/conv_tune.txt (the B200-tuned kernel configurations every
    bench / test run imports) parses completely -- a line the parser rejected
    would silently fall back to run-time tuning -- holds every shape of the
    headline step (k = 42: fwd / dgrad / wgrad of the ResNet-152 convs), and
    exports back unchanged.  Host-only code: no GPU needed."""
    text = open(os.path.join(ROOT, "profiles", "b200", "conv_tune.txt")).read()
    lines = sorted(l.strip() for l in text.splitlines() if l.strip())
    for l in lines:
        v = [int(t) for t in l.split()]
        assert len(v) in (18, 19), l
        bn, splits, cm = v[14], v[15], v[16]
        assert bn in (64, 128, 256) and splits >= 1 and cm in (1, 2, 4, 5, 6, 7, 8), l
    assert sum(1 for l in lines if l.split()[1] == "42") >= 70
    _native.conv_tune_import(text)
    assert sorted(_native.conv_tune_export().splitlines()) == lines
