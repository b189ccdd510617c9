"""Loader for the in-tree native libraries.

The libraries are built in-tree by ``__graft_entry__.build()`` (csrc/Makefile)
into ``paper_1901_06773_b200/lib``.  There is no CPU or eager fallback: if a
library is missing, every entry point raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")
PLANNER_LIB = os.path.join(LIB_DIR, "libswapsched_b200.so")
CUDA_LIB = os.path.join(LIB_DIR, "libaccudnn.so")

_planner = None
_cuda = None


class NativeMissing(RuntimeError):
    pass


def planner_lib():
    """libswapsched_b200.so (host planner; loads without a GPU)."""
    global _planner
    if _planner is None:
        if not os.path.exists(PLANNER_LIB):
            raise NativeMissing(f"{PLANNER_LIB} not built; run __graft_entry__.build()")
        lib = ctypes.CDLL(PLANNER_LIB)
        _declare_planner(lib)
        _planner = lib
    return _planner


def cuda_lib():
    """libaccudnn.so (sm_100a kernels + executor)."""
    global _cuda
    if _cuda is None:
        if not os.path.exists(CUDA_LIB):
            raise NativeMissing(f"{CUDA_LIB} not built; run __graft_entry__.build()")
        planner_lib()  # dependency, resolved through rpath as well
        # torch first: its bundled libnccl.so.2 (2.28) must be the one the
        # process maps; libaccudnn's NEEDED libnccl.so.2 then binds to it
        # instead of the older system copy torch cannot run with.
        import torch  # noqa: F401
        lib = ctypes.CDLL(CUDA_LIB)
        _declare_cuda(lib)
        _cuda = lib
    return _cuda


c_char_pp = ctypes.POINTER(ctypes.c_char_p)


class PlanOpts(ctypes.Structure):
    _fields_ = [
        ("step", ctypes.c_int),
        ("k_override", ctypes.c_int),
        ("epochs", ctypes.c_longlong),
        ("dataset_size", ctypes.c_longlong),
        ("budget_override", ctypes.c_ulonglong),
    ]


class ConvDesc(ctypes.Structure):
    _fields_ = [(name, ctypes.c_int) for name in
                ("n", "h", "w", "c", "k", "r", "s", "stride", "pad", "p", "q")]


PLANNER_SYMBOLS = {
    "last_error": ([], ctypes.c_char_p),
    "free": ([ctypes.c_void_p], None),
    "validate": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "fit": ([ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, ctypes.c_char_p,
             ctypes.c_double, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "kmax": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "plan": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(PlanOpts),
              ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "evaluate_k": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int,
                    ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "simulate": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                  ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                  ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "phase_times": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
                    ctypes.c_int),
    "simulate_report": ([ctypes.c_char_p] * 5 + [ctypes.c_int, ctypes.c_ulonglong, ctypes.c_double]
                        + [ctypes.POINTER(ctypes.c_void_p)] * 5, ctypes.c_int),
    "with_digest": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)],
                    ctypes.c_int),
    "sweep": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int),
               ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
              ctypes.c_int),
    "tune_lr": ([ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                 ctypes.c_longlong, ctypes.POINTER(ctypes.c_double),
                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong)],
                ctypes.c_int),
    "generate_fixture": ([ctypes.c_ulonglong, ctypes.c_int, ctypes.c_int] +
                         [ctypes.POINTER(ctypes.c_void_p)] * 4, ctypes.c_int),
}


def declare_planner_symbols(lib, prefix):
    for name, (args, res) in PLANNER_SYMBOLS.items():
        fn = getattr(lib, prefix + name)
        fn.argtypes = args
        fn.restype = res


def _declare_planner(lib):
    declare_planner_symbols(lib, "accudnn_")


_P = ctypes.c_void_p
_I = ctypes.c_int
_LL = ctypes.c_longlong
_F = ctypes.c_float

CUDA_SYMBOLS = {
    "accudnn_set_conv_math": ([_I], _I),
    "accudnn_get_conv_math": ([], _I),
    "accudnn_set_conv_impl": ([_I], _I),
    "accudnn_conv_set_workspace": ([ctypes.c_void_p, ctypes.c_ulonglong], _I),
    "accudnn_conv_set_precise_scratch": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_ulonglong], _I),
    "accudnn_conv_precise_scratch_bytes": ([_P], ctypes.c_ulonglong),
    "accudnn_conv_set_stream_workspace": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_ulonglong, _I], _I),
    "accudnn_conv_autotune": ([_I], _I),
    "accudnn_conv_tune_export": ([ctypes.POINTER(ctypes.c_void_p)], _I),
    "accudnn_conv_tune_import": ([ctypes.c_char_p], _I),
    "accudnn_conv_force_cfg": ([_I, _I, _I], _I),
    "accudnn_set_pdl": ([_I], _I),
    "accudnn_conv_trace": ([_P], _I),
    "accudnn_bn_trace": ([_P], _I),
    "accudnn_conv_fwd": ([ctypes.POINTER(ConvDesc), _P, _P, _P, _I, _P], _I),
    "accudnn_conv_dgrad": ([ctypes.POINTER(ConvDesc), _P, _P, _P, _I, _P], _I),
    "accudnn_conv_fwd_stats": ([ctypes.POINTER(ConvDesc), _P, _P, _P, _P, ctypes.POINTER(_I), _P], _I),
    "accudnn_conv_wgrad": ([ctypes.POINTER(ConvDesc), _P, _P, _P, _I, _I, _P], _I),
    "accudnn_bn_workspace_bytes": ([_I], ctypes.c_ulonglong),
    "accudnn_bn_fwd": ([_P, _LL, _I, _P, _P, _F, _I, _P, _P, _P, _P, _P, _F, _P, _P], _I),
    "accudnn_bn_bwd": ([_P, _P, _LL, _I, _P, _P, _P, _P, _I, _P, _I, _P, _P, _P, _P], _I),
    "accudnn_bn_fwd_stats": ([_P, _P, _LL, _I, _P, _P, _F, _I, _P, _P, _P, _P, _P, _F, _P, _P], _I),
    "accudnn_bn_add_relu_fwd_stats": ([_P, _P, _P, _LL, _I, _P, _P, _F, _P, _P, _P, _P, _P, _F, _P,
                                       _P], _I),
    "accudnn_bn_add_relu_fwd": ([_P, _P, _LL, _I, _P, _P, _F, _P, _P, _P, _P, _P, _F, _P, _P], _I),
    "accudnn_bn_add_relu_bwd": ([_P, _P, _P, _LL, _I, _P, _P, _P, _P, _P, _I, _P, _I, _P, _P, _P,
                                 _P], _I),
    "accudnn_bn_relu_apply": ([_P, ctypes.c_longlong, _I, _P, _P, _P, _P, _P, _P], _I),
    "accudnn_relu_fwd": ([_P, _P, _LL, _P], _I),
    "accudnn_relu_bwd": ([_P, _P, _P, _LL, _I, _P], _I),
    "accudnn_add_fwd": ([_P, _P, _P, _LL, _P], _I),
    "accudnn_copy": ([_P, _P, _LL, _I, _P], _I),
    "accudnn_maxpool_fwd": ([_P] + [_I] * 10 + [_P, _P], _I),
    "accudnn_maxpool_bwd": ([_P, _P] + [_I] * 10 + [_P, _P], _I),
    "accudnn_avgpool_fwd": ([_P, _I, _I, _I, _P, _P], _I),
    "accudnn_avgpool_bwd": ([_P, _I, _I, _I, _P, _P], _I),
    "accudnn_bias_add": ([_P, _P, _LL, _I, _P], _I),
    "accudnn_xent_fwd": ([_P, _P, _I, _I, _P, _P], _I),
    "accudnn_xent_bwd": ([_P, _P, _I, _I, _P, _P, _P], _I),
    "accudnn_sgd_update": ([_P, _P, _P, _LL, _F, _F, _F, _F, _I, _P], _I),
    "accudnn_nchw_to_nhwc_pad": ([_P, _I, _I, _I, _I, _I, _P, _P], _I),
}


def _declare_cuda(lib):
    for name, (args, res) in CUDA_SYMBOLS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    try:
        from . import _exec_symbols
        _exec_symbols.declare(lib)
    except ImportError:
        pass


def conv_tune_export():
    """the conv autotuner's table (text, see include/accudnn_kernels.h)"""
    import ctypes as _c
    lib = cuda_lib()
    p = _c.c_void_p()
    if lib.accudnn_conv_tune_export(_c.byref(p)) != 0:
        raise RuntimeError("accudnn_conv_tune_export failed")
    try:
        return _c.string_at(p).decode()
    finally:
        _c.CDLL(None).free(p)


def conv_tune_import(text):
    if cuda_lib().accudnn_conv_tune_import(text.encode()) != 0:
        raise RuntimeError("accudnn_conv_tune_import failed")
