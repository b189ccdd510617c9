"""Python mirror of the reference planner/tuner entry points.

Each function is one document-level operation of the reference CLI
(/root/reference/proj/tools/swapsched.cpp), executed by the bit-exact host
C++ restatement in libswapsched_b200.so through the C ABI declared in
include/accudnn_plan.h.  Errors follow the CLI's exit-code contract
(swapsched.cpp:654-672): ``PlannerError.code`` is 1 for validation /
infeasible / untrainable, 2 for I/O, 3 for internal errors.

The same functions can drive the compiled reference oracle (tests only) by
passing ``lib=`` and ``prefix="oracle_"``.
"""

import ctypes
import json
import os

from . import _native


class PlannerError(RuntimeError):
    def __init__(self, code, message, document=None):
        super().__init__(f"[exit {code}] {message}")
        self.code = code
        self.message = message
        self.document = document


class _Binding:
    def __init__(self, lib=None, prefix="accudnn_"):
        self.lib = lib if lib is not None else _native.planner_lib()
        self.prefix = prefix

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def take(self, ptr):
        if not ptr:
            return None
        text = ctypes.string_at(ptr).decode()
        self.fn("free")(ptr)
        return text

    def error(self):
        msg = self.fn("last_error")()
        return msg.decode() if msg else ""


def _b(s):
    return s.encode() if isinstance(s, str) else s


def _docs(*docs):
    return [_b(d if isinstance(d, str) or d is None else json.dumps(d)) for d in docs]


def validate(network_json, *, lib=None, prefix="accudnn_"):
    """GMAP diagnostics (``swapsched validate``); returns the report text."""
    B = _Binding(lib, prefix)
    out = ctypes.c_void_p()
    rc = B.fn("validate")(*_docs(network_json), ctypes.byref(out))
    text = B.take(out.value)
    if rc not in (0, 1) or (rc == 1 and not text):
        raise PlannerError(rc, B.error())
    return rc, text


def fit(network_json, profile_csvs, hardware_json=None, eta=0.95, *, lib=None,
        prefix="accudnn_"):
    """Fit model.json from compute/transfer profile CSV texts (``swapsched fit``)."""
    B = _Binding(lib, prefix)
    arr = (ctypes.c_char_p * len(profile_csvs))(*[_b(t) for t in profile_csvs])
    out = ctypes.c_void_p()
    rc = B.fn("fit")(_docs(network_json)[0], arr, len(profile_csvs),
                     _docs(hardware_json)[0] if hardware_json is not None else None,
                     float(eta), ctypes.byref(out))
    text = B.take(out.value)
    if rc != 0:
        raise PlannerError(rc, B.error())
    return text


def kmax(network_json, hardware_json, *, lib=None, prefix="accudnn_"):
    B = _Binding(lib, prefix)
    k = ctypes.c_int(0)
    rc = B.fn("kmax")(*_docs(network_json, hardware_json), ctypes.byref(k))
    if rc != 0:
        raise PlannerError(rc, B.error())
    return k.value


def plan(network_json, hardware_json, model_json, *, step=1, k_override=0, epochs=1,
         dataset_size=0, budget_override=0, lib=None, prefix="accudnn_"):
    """Algorithm 2 + greedy pinning (``swapsched plan``); returns plan.json text.

    Raises PlannerError(code=1) with the status document when the budget is
    untrainable or no minibatch satisfies the stall constraint.
    """
    B = _Binding(lib, prefix)
    opts = _native.PlanOpts(step, k_override, epochs, dataset_size, budget_override)
    out = ctypes.c_void_p()
    rc = B.fn("plan")(*_docs(network_json, hardware_json, model_json), ctypes.byref(opts),
                      ctypes.byref(out))
    text = B.take(out.value)
    if rc != 0:
        raise PlannerError(rc, B.error(), text)
    return text


def phase_times(network_json, model_json, k, *, lib=None, prefix="accudnn_"):
    """The model's 2N phase compute times at k, in integer ns (list)."""
    B = _Binding(lib, prefix)
    out = ctypes.c_void_p()
    rc = B.fn("phase_times")(_b(network_json), _b(model_json), int(k), ctypes.byref(out))
    text = B.take(out.value)
    if rc != 0:
        raise PlannerError(rc, B.error())
    return [int(line.split(",")[1]) for line in text.splitlines()[1:]]


class PlanSession:
    """Incremental re-planning (accudnn_plan_session_*): the documents are
    parsed once and everything Algorithm 2 derives per k independently of
    the device cap and the host-link bandwidth is cached, so re-plans for a
    new cap / bandwidth reuse it.  plan() returns what plan() above returns
    for the changed documents; exact=True answers any step with the
    step-1 scan."""

    def __init__(self, network_json, hardware_json, model_json):
        lib = _native.planner_lib()
        self._lib = lib
        lib.accudnn_plan_session_create.argtypes = [ctypes.c_char_p] * 3 + [
            ctypes.POINTER(ctypes.c_void_p)]
        lib.accudnn_plan_session_plan.argtypes = [
            ctypes.c_void_p, ctypes.POINTER(_native.PlanOpts), ctypes.c_double, ctypes.c_int,
            ctypes.POINTER(ctypes.c_void_p)]
        lib.accudnn_plan_session_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong),
                                                   ctypes.POINTER(ctypes.c_longlong)]
        lib.accudnn_plan_session_destroy.argtypes = [ctypes.c_void_p]
        lib.accudnn_plan_session_destroy.restype = None
        lib.accudnn_session_last_error.restype = ctypes.c_char_p
        h = ctypes.c_void_p()
        rc = lib.accudnn_plan_session_create(*_docs(network_json, hardware_json, model_json),
                                             ctypes.byref(h))
        if rc != 0:
            raise PlannerError(rc, lib.accudnn_session_last_error().decode())
        self._h = h

    def plan(self, *, budget_override=0, bandwidth=0.0, step=1, k_override=0, epochs=1,
             dataset_size=0, exact=False):
        opts = _native.PlanOpts(step, k_override, epochs, dataset_size, budget_override)
        out = ctypes.c_void_p()
        rc = self._lib.accudnn_plan_session_plan(self._h, ctypes.byref(opts), float(bandwidth),
                                                 1 if exact else 0, ctypes.byref(out))
        text = None
        if out.value:
            text = ctypes.string_at(out.value).decode()
            self._lib.accudnn_free(out.value)
        if rc != 0:
            raise PlannerError(rc, self._lib.accudnn_session_last_error().decode(), text)
        return text

    def stats(self):
        hits, misses = ctypes.c_longlong(), ctypes.c_longlong()
        self._lib.accudnn_plan_session_stats(self._h, ctypes.byref(hits), ctypes.byref(misses))
        return {"hits": hits.value, "misses": misses.value}

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.accudnn_plan_session_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def evaluate_k(network_json, hardware_json, model_json, k, *, lib=None, prefix="accudnn_"):
    """One evaluate_minibatch (integer-ns t_ready, pin names) as a dict."""
    B = _Binding(lib, prefix)
    out = ctypes.c_void_p()
    rc = B.fn("evaluate_k")(*_docs(network_json, hardware_json, model_json), int(k),
                            ctypes.byref(out))
    text = B.take(out.value)
    if rc != 0:
        raise PlannerError(rc, B.error())
    return json.loads(text)


def simulate(network_json, hardware_json, model_json, plan_json=None, mode="dynamic", k=0,
             *, lib=None, prefix="accudnn_"):
    """Three-stream iteration model (``swapsched simulate``).

    Returns (rc, summary_json_text, trace_csv_text); rc 1 means the
    simulated iteration deadlocked (summary carries oom_detail)."""
    B = _Binding(lib, prefix)
    summ, trace = ctypes.c_void_p(), ctypes.c_void_p()
    rc = B.fn("simulate")(*_docs(network_json, hardware_json, model_json),
                          _b(plan_json) if plan_json is not None else None, _b(mode), int(k),
                          ctypes.byref(summ), ctypes.byref(trace))
    s, t = B.take(summ.value), B.take(trace.value)
    if rc not in (0, 1) or s is None:
        raise PlannerError(rc, B.error())
    return rc, s, t


def simulate_report(network_json, hardware_json, model_json, plan_json=None, mode="dynamic",
                    k=0, budget_override=0, tolerance=0.02, *, lib=None, prefix="accudnn_"):
    """Everything ``swapsched simulate`` writes (swapsched.cpp:300-383).

    Returns (rc, dict) with keys summary, trace, mem_curves, stall_bars and
    verify (the verify_plan document, "" without a plan); rc 1 means a
    deadlocked iteration or a failed verdict."""
    B = _Binding(lib, prefix)
    outs = [ctypes.c_void_p() for _ in range(5)]
    rc = B.fn("simulate_report")(*_docs(network_json, hardware_json, model_json),
                                 _b(plan_json) if plan_json is not None else None, _b(mode),
                                 int(k), int(budget_override), float(tolerance),
                                 *[ctypes.byref(o) for o in outs])
    texts = [B.take(o.value) for o in outs]
    if rc not in (0, 1) or texts[0] is None:
        raise PlannerError(rc, B.error())
    keys = ("summary", "trace", "mem_curves", "stall_bars", "verify")
    return rc, dict(zip(keys, texts))


def with_digest(doc, digest, *, lib=None, prefix="accudnn_"):
    """The document with "manifest_digest" added, serialised exactly as the
    reference CLI writes it (swapsched.cpp:114-118)."""
    B = _Binding(lib, prefix)
    out = ctypes.c_void_p()
    rc = B.fn("with_digest")(_b(doc), _b(digest), ctypes.byref(out))
    text = B.take(out.value)
    if rc != 0:
        raise PlannerError(rc, B.error())
    return text


def sweep(network_json, hardware_json, model_json, ks, modes="naive,dynamic,resident",
          parallel=True, *, lib=None, prefix="accudnn_"):
    B = _Binding(lib, prefix)
    arr = (ctypes.c_int * len(ks))(*ks)
    out = ctypes.c_void_p()
    rc = B.fn("sweep")(*_docs(network_json, hardware_json, model_json), arr, len(ks),
                       _b(modes), 1 if parallel else 0, ctypes.byref(out))
    text = B.take(out.value)
    if rc != 0:
        raise PlannerError(rc, B.error())
    return text


def tune_lr(alpha_base, convexity, q, mu=1.0, iters_base=1000, *, lib=None,
            prefix="accudnn_"):
    """Eq. 9 learning rate (``swapsched tune-lr``): (alpha*, residual, iterations)."""
    B = _Binding(lib, prefix)
    a, r, it = ctypes.c_double(), ctypes.c_double(), ctypes.c_longlong()
    rc = B.fn("tune_lr")(float(alpha_base), float(convexity), float(mu), float(q),
                         int(iters_base), ctypes.byref(a), ctypes.byref(r), ctypes.byref(it))
    if rc != 0:
        raise PlannerError(rc, B.error())
    return a.value, r.value, it.value


def generate_fixture(seed, min_layers=0, max_layers=0, *, lib=None, prefix="accudnn_"):
    """Seeded synthetic instance (``swapsched gen``): dict of the four documents."""
    B = _Binding(lib, prefix)
    outs = [ctypes.c_void_p() for _ in range(4)]
    rc = B.fn("generate_fixture")(int(seed), int(min_layers), int(max_layers),
                                  *[ctypes.byref(o) for o in outs])
    texts = [B.take(o.value) for o in outs]
    if rc != 0:
        raise PlannerError(rc, B.error())
    return dict(zip(("network", "hardware", "compute_csv", "transfer_csv"), texts))


def _fnv1a(chunks):
    h = 1469598103934665603
    for data in chunks:
        for c in data:
            h ^= c
            h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def plan_cached(network_json, hardware_json, model_json, cache_dir, *, step=1, k_override=0,
                epochs=1, dataset_size=0, budget_override=0, lib=None, prefix="accudnn_"):
    """plan() behind a persistent cache keyed by the reference's manifest
    digest of the `plan` run (FNV-1a over the subcommand, the three documents
    and the `key=value;` parameters, swapsched.cpp:76-91): the same inputs
    return the stored plan.json without re-planning.  Returns (plan_json, hit)."""
    params = [("step", step), ("k", k_override), ("epochs", epochs),
              ("dataset_size", dataset_size)]
    if budget_override:
        params.append(("budget", budget_override))
    digest = _fnv1a([b"plan", _b(network_json), _b(hardware_json), _b(model_json)] +
                    [f"{k}={v};".encode() for k, v in params])
    path = os.path.join(cache_dir, f"plan-{digest}.json")
    if os.path.exists(path):
        with open(path) as f:
            return f.read(), True
    text = plan(network_json, hardware_json, model_json, step=step, k_override=k_override,
                epochs=epochs, dataset_size=dataset_size, budget_override=budget_override,
                lib=lib, prefix=prefix)
    os.makedirs(cache_dir, exist_ok=True)
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        f.write(text)
    os.replace(tmp, path)
    return text, False
