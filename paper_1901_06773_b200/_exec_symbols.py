"""ctypes declarations for include/accudnn.h (executor C ABI)."""
import ctypes

_P = ctypes.c_void_p
_I = ctypes.c_int
_LL = ctypes.c_longlong
_F = ctypes.c_float
_S = ctypes.c_char_p
_ULLP = ctypes.POINTER(ctypes.c_ulonglong)


class StepStats(ctypes.Structure):
    _fields_ = [("loss", ctypes.c_float), ("iter_ms", ctypes.c_double),
                ("exposed_swap_ms", ctypes.c_double), ("allreduce_ms", ctypes.c_double),
                ("peak_bytes", ctypes.c_ulonglong), ("swapped_bytes", ctypes.c_ulonglong),
                ("exposed_allreduce_ms", ctypes.c_double)]


SYMBOLS = {
    "accudnn_rt_last_error": ([], _S),
    "accudnn_rt_free": ([_P], None),
    "accudnn_net_export": ([_S, _I, _I, _I, _I, ctypes.POINTER(_P), ctypes.POINTER(_P)], _I),
    "accudnn_net_memory": ([_S, _I, _I, _I, _I, _P, ctypes.POINTER(_LL), ctypes.POINTER(_LL)], _I),
    "accudnn_exec_create": ([_S, _I, _I, _S, _S, _S, _S, _I, _I, _I, ctypes.POINTER(_P)], _I),
    "accudnn_exec_destroy": ([_P], _I),
    "accudnn_exec_num_params": ([_P], _LL),
    "accudnn_exec_num_stats": ([_P], _LL),
    "accudnn_exec_set_params": ([_P, _P, _LL], _I),
    "accudnn_exec_get_params": ([_P, _P, _LL], _I),
    "accudnn_exec_get_grads": ([_P, _P, _LL], _I),
    "accudnn_exec_get_stats": ([_P, _P, _LL], _I),
    "accudnn_exec_set_graph": ([_P, _I], _I),
    "accudnn_exec_step": ([_P, _P, _P, _I, _F, _I, _I, ctypes.POINTER(StepStats)], _I),
    "accudnn_exec_step_pipelined": ([_P, _P, _P, _F, _I, _P, ctypes.POINTER(StepStats)], _I),
    "accudnn_exec_memory": ([_P, _ULLP, _ULLP], _I),
    "accudnn_exec_launches": ([_P], _I),
    "accudnn_exec_trace": ([_P, ctypes.POINTER(_P)], _I),
    "accudnn_exec_document": ([_P, _S, ctypes.POINTER(_P)], _I),
    "accudnn_nccl_unique_id": ([_P], _I),
    "accudnn_exec_set_comm": ([_P, _P, _I, _I], _I),
    "accudnn_exec_comm_bytes": ([_P], ctypes.c_ulonglong),
}


def declare(lib):
    for name, (args, res) in SYMBOLS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
