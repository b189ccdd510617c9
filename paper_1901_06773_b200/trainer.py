"""Host-side mirror of the training step: network export, executor, one
SGD step per call.

Everything runs in libaccudnn.so (include/accudnn.h); this module only
marshals arguments.  There is no fallback path: a missing library or a
failing CUDA call raises.
"""

import ctypes
import json

import numpy as np

from . import _native
from ._exec_symbols import StepStats


class ExecutorError(RuntimeError):
    pass


def _lib():
    return _native.cuda_lib()


def _take(ptr):
    if not ptr:
        return None
    s = ctypes.string_at(ptr).decode()
    _lib().accudnn_rt_free(ptr)
    return s


def _check(rc, what):
    if rc != 0:
        msg = _lib().accudnn_rt_last_error()
        raise ExecutorError(f"{what} failed (rc={rc}): {msg.decode() if msg else ''}")


def export_network(arch, image, classes, k_base=8, lookahead=1):
    """(network.json text, op description dict) of an architecture.

    network.json follows the reference format (model_ir.cpp:87-144): one
    LayerDecl per executed op, featuremap = the op's output, workspace =
    every other byte the executor holds in that layer's phases."""
    a, b = ctypes.c_void_p(), ctypes.c_void_p()
    _check(_lib().accudnn_net_export(arch.encode(), int(image), int(classes), int(k_base),
                                     int(lookahead), ctypes.byref(a), ctypes.byref(b)),
           "net export")
    return _take(a.value), json.loads(_take(b.value))


def net_memory(arch, image, classes, k, swapped, lookahead=1):
    """(peak live bytes, static arena bytes) of the executor's tensor
    instances for a swap mask -- computed on the host, no GPU needed."""
    mask = (ctypes.c_char * len(swapped))(*[b"\x01" if s else b"\x00" for s in swapped])
    live, arena = ctypes.c_longlong(), ctypes.c_longlong()
    _check(_lib().accudnn_net_memory(arch.encode(), int(image), int(classes), int(k),
                                     int(lookahead), mask, ctypes.byref(live),
                                     ctypes.byref(arena)), "net memory")
    return live.value, arena.value


def hardware_json(budget_bytes, m_others_bytes, pcie_bytes_per_s, delta_sync_s=0.0):
    return json.dumps({"format_version": 1, "memory_budget_bytes": int(budget_bytes),
                       "m_others_bytes": int(m_others_bytes), "delta_sync_s": float(delta_sync_s),
                       "pcie_nominal_bytes_per_s": float(pcie_bytes_per_s)}, indent=2) + "\n"


def default_m_others(describe, image, budget_bytes=None):
    """Fixed device bytes outside params+grads: the momentum buffer, BN
    statistics and a staging allowance for the input batch (the paper's
    "pre-cached inputs and fixed overheads").  The executor keeps
    the batch twice (NCHW staging + NHWC4 for the stem, 7 floats per pixel);
    with a budget the allowance covers the largest batch the budget could
    hold at all (budget / featuremap bytes per image), so a tuned k* always
    fits the executor's fixed allocations.  What the batch leaves of it is
    the convolutions' split-K workspace (shared by the compute and the
    weight-gradient streams)."""
    momentum = 4 * describe["n_params"]
    stats = 4 * describe["n_stats"]
    staging = (96 << 20) if image >= 128 else (32 << 20)
    if budget_bytes:
        fm_per_image = sum(4 * o["out"][0] * o["out"][1] * o["out"][2] for o in describe["ops"]
                           if not o.get("transient"))
        k_ub = int(budget_bytes) // max(1, fm_per_image)
        staging = max(staging, 7 * 4 * image * image * k_ub + (8 << 20))
    return momentum + stats + staging


def precise_scratch_allowance(describe, image, budget_bytes):
    """Fixed device bytes of the 3xTF32 mode (accudnn_set_conv_math(1)): the
    executor's scratch for the operands' low parts of its largest
    convolution (max over fwd / dgrad / wgrad of the two operands' bytes,
    accudnn_conv_precise_scratch_bytes), at the largest batch the budget
    could hold at all (as default_m_others sizes the input staging)."""
    ops = describe["ops"]
    fm_per_image = sum(4 * o["out"][0] * o["out"][1] * o["out"][2] for o in ops
                       if not o.get("transient"))
    k_ub = max(1, int(budget_bytes) // max(1, fm_per_image))
    by_id = {o["id"]: o for o in ops}
    worst = 0
    for o in ops:
        if o["kind"] not in ("conv", "fc"):
            continue
        src = by_id.get(o["in0"])
        xin = (image * image * o["cin"]) if src is None else \
            src["out"][0] * src["out"][1] * src["out"][2]
        if o["kind"] == "fc":
            xin = o["cin"]
        yout = o["out"][0] * o["out"][1] * o["out"][2] if o["kind"] == "conv" else o["cout"]
        w = o["cout"] * o["cin"] * o.get("r", 1) ** 2
        x, y = 4 * xin * k_ub, 4 * yout * k_ub
        worst = max(worst, x + 4 * w, y + 4 * w, x + y)
    return worst + (4 << 20)  # 256-byte alignment of the two parts and slack


def config_documents(arch, image, classes, cap_bytes, k_base=8):
    """The planner's input documents for one BASELINE configuration, exactly
    as bench.py and the headline plan goldens build them: network.json from
    the exporter, hardware.json (cap, fixed overhead, measured host-link
    bandwidth from profiles/b200/host_link.json) and model.json fitted
    (eta = 0.95) from the committed B200 profile CSVs.  Returns
    (network_json, hardware_json, model_json, describe)."""
    import os

    from . import planner
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pdir = os.path.join(root, "profiles", "b200")
    network_json, desc = export_network(arch, image, classes, k_base=k_base)
    link = {}
    lp = os.path.join(pdir, "host_link.json")
    if os.path.exists(lp):
        link = json.load(open(lp))
    pcie = float(link.get("d2h", 50.0)) * 1e9
    m_others = default_m_others(desc, image, int(cap_bytes))
    hw = hardware_json(int(cap_bytes), m_others, pcie)
    csvs = [open(os.path.join(pdir, f"{arch}_{kind}_profile.csv")).read()
            for kind in ("compute", "transfer")]
    model_json = planner.fit(network_json, csvs, hw, eta=0.95)
    return network_json, hw, model_json, desc


def init_params(describe, seed=0):
    """torchvision-style initialisation of the flat parameter vector:
    Kaiming-normal (fan_out, ReLU) convs, BN gamma=1 / beta=0, FC uniform
    +-1/sqrt(fan_in)."""
    rng = np.random.default_rng(seed)
    p = np.zeros(describe["n_params"], dtype=np.float32)
    for op in describe["ops"]:
        if op["kind"] == "conv":
            cout, cin, r = op["cout"], op["cin"], op["r"]
            std = (2.0 / (cout * r * r)) ** 0.5
            w = rng.standard_normal((cout, r, r, cin)).astype(np.float32) * std
            if op["in0"] == -2:  # zero the padded input channel
                w[..., describe["in_channels"]:] = 0.0
            p[op["w_off"]:op["w_off"] + w.size] = w.ravel()
        elif op["kind"] == "fc":
            cout, cin = op["cout"], op["cin"]
            bound = 1.0 / cin ** 0.5
            p[op["w_off"]:op["w_off"] + cout * cin] = rng.uniform(-bound, bound, cout * cin)
            p[op["b_off"]:op["b_off"] + cout] = rng.uniform(-bound, bound, cout)
        elif op["kind"] in ("bn", "bn_relu", "bn_add_relu"):
            c = op["channels"]
            p[op["g_off"]:op["g_off"] + c] = 1.0
            p[op["beta_off"]:op["beta_off"] + c] = 0.0
    return p


class Executor:
    """One training-step executor on one GPU (include/accudnn.h).

    mode: "resident" | "naive" | "dynamic" (plan_json's pin set)."""

    def __init__(self, arch, image, classes, k=0, mode="resident", plan_json=None,
                 network_json=None, hardware_json=None, device=0, lookahead=1):
        self.lib = _lib()
        self.arch, self.image, self.classes = arch, image, classes
        h = ctypes.c_void_p()
        enc = lambda s: s.encode() if isinstance(s, str) else s  # noqa: E731
        _check(self.lib.accudnn_exec_create(arch.encode(), int(image), int(classes), enc(mode),
                                            enc(network_json), enc(hardware_json),
                                            enc(plan_json), int(k), int(device), int(lookahead),
                                            ctypes.byref(h)), "executor create")
        self.h = h
        self.device = int(device)
        if k <= 0:
            k = json.loads(plan_json)["k_star"]
        self.k = k
        self.n_params = self.lib.accudnn_exec_num_params(h)
        self.n_stats = self.lib.accudnn_exec_num_stats(h)

    def close(self):
        if self.h:
            self.lib.accudnn_exec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_params(self, flat):
        flat = np.ascontiguousarray(flat, dtype=np.float32)
        _check(self.lib.accudnn_exec_set_params(self.h, flat.ctypes.data, flat.size), "set_params")

    def _get(self, fn, n):
        out = np.empty(n, dtype=np.float32)
        _check(fn(self.h, out.ctypes.data, n), "copy out")
        return out

    def get_params(self):
        return self._get(self.lib.accudnn_exec_get_params, self.n_params)

    def get_grads(self):
        return self._get(self.lib.accudnn_exec_get_grads, self.n_params)

    def get_stats(self):
        return self._get(self.lib.accudnn_exec_get_stats, self.n_stats)

    def set_graph(self, enable=True):
        self.lib.accudnn_exec_set_graph(self.h, 1 if enable else 0)

    def memory(self):
        a, f = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        self.lib.accudnn_exec_memory(self.h, ctypes.byref(a), ctypes.byref(f))
        return a.value, f.value

    def launches(self):
        return self.lib.accudnn_exec_launches(self.h)

    def trace(self):
        p = ctypes.c_void_p()
        _check(self.lib.accudnn_exec_trace(self.h, ctypes.byref(p)), "trace")
        return _take(p.value)

    def _check_batch(self, images, labels):
        """The kernels read images as contiguous float32 NCHW [k,3,H,W] and
        labels as contiguous int32 [k] in [0, classes): anything else is
        rejected here rather than reinterpreted (torch's default int64 labels
        would read as (low, high) int32 pairs)."""
        shape = (self.k, 3, self.image, self.image)
        for name, a, dt, shp in (("images", images, "float32", shape),
                                 ("labels", labels, "int32", (self.k,))):
            if a is None:
                continue
            if hasattr(a, "data_ptr"):  # torch tensor
                ok = str(a.dtype) == "torch." + dt and a.is_contiguous()
                if a.is_cuda and a.device.index != self.device:
                    raise ExecutorError(f"{name} on cuda:{a.device.index}, executor on cuda:{self.device}")
            else:
                ok = a.dtype == np.dtype(dt) and a.flags["C_CONTIGUOUS"]
            if not ok or tuple(a.shape) != shp:
                raise ExecutorError(f"{name}: need contiguous {dt} {list(shp)}, got "
                                    f"{a.dtype} {list(a.shape)}")
        if labels is not None and not (hasattr(labels, "is_cuda") and labels.is_cuda):
            lo, hi = int(labels.min()), int(labels.max())
            if lo < 0 or hi >= self.classes:
                raise ExecutorError(f"labels outside [0, {self.classes}): [{lo}, {hi}]")

    def document(self, which):
        """reference-schema documents of the last profiled step: "trace",
        "mem_curves", "stall_bars", "summary"; "order" = copies in stream order"""
        p = ctypes.c_void_p()
        _check(self.lib.accudnn_exec_document(self.h, which.encode(), ctypes.byref(p)), "document")
        return _take(p.value)

    def step(self, images, labels, lr=0.1, update=True, profile=False):
        """images: NCHW float32 [k,3,H,W]; labels int32 [k].  numpy arrays (or
        CPU torch tensors) are copied from host memory inside the step; CUDA
        torch tensors are used in place (a device label outside [0, classes)
        makes the loss NaN)."""
        host = 1
        if not hasattr(images, "data_ptr"):
            images = np.asarray(images)
            labels = np.asarray(labels)
        self._check_batch(images, labels)
        if hasattr(images, "is_cuda") and images.is_cuda:
            if not labels.is_cuda:
                raise ExecutorError("images on the device need device labels")
            host = 0
            ip, lp = images.data_ptr(), labels.data_ptr()
        elif hasattr(images, "data_ptr"):
            ip, lp = images.data_ptr(), labels.data_ptr()
        else:
            ip, lp = images.ctypes.data, labels.ctypes.data
        st = StepStats()
        _check(self.lib.accudnn_exec_step(self.h, ip, lp, host, float(lr), 1 if update else 0,
                                          1 if profile else 0, ctypes.byref(st)), "step")
        return {"loss": st.loss, "iter_ms": st.iter_ms, "exposed_swap_ms": st.exposed_swap_ms,
                "peak_bytes": st.peak_bytes, "swapped_bytes": st.swapped_bytes,
                "allreduce_ms": st.allreduce_ms, "exposed_allreduce_ms": st.exposed_allreduce_ms}

    def step_pipelined(self, images, labels, lr=0.1, update=True, next_images=None):
        """host-input step with the next batch's H2D overlapped: images=None
        uses the batch prefetched by the previous call; next_images (pinned
        host tensor / array) is prefetched during this step."""
        keep = []  # converted arrays must outlive the (synchronous) call
        self._check_batch(images, labels)
        if next_images is not None:
            self._check_batch(next_images, None)

        def ptr(a, dtype=np.float32):
            if a is None:
                return None
            if hasattr(a, "data_ptr"):
                return a.data_ptr()
            keep.append(np.ascontiguousarray(a, dtype=dtype))
            return keep[-1].ctypes.data
        lp = ptr(labels, np.int32)
        st = StepStats()
        _check(self.lib.accudnn_exec_step_pipelined(self.h, ptr(images), lp, float(lr),
                                                    1 if update else 0, ptr(next_images),
                                                    ctypes.byref(st)), "step")
        return {"loss": st.loss, "iter_ms": st.iter_ms, "exposed_swap_ms": st.exposed_swap_ms,
                "peak_bytes": st.peak_bytes, "swapped_bytes": st.swapped_bytes,
                "allreduce_ms": st.allreduce_ms, "exposed_allreduce_ms": st.exposed_allreduce_ms}

    def set_comm(self, uid_bytes, rank, world):
        buf = ctypes.create_string_buffer(bytes(uid_bytes), 128)
        _check(self.lib.accudnn_exec_set_comm(self.h, buf, int(rank), int(world)), "set_comm")

    def comm_bytes(self):
        """device bytes NCCL allocated for this executor's communicator"""
        return self.lib.accudnn_exec_comm_bytes(self.h)


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(_lib().accudnn_nccl_unique_id(buf), "ncclGetUniqueId")
    return buf.raw
