"""Host-link transfer microbenchmark: copy-engine cudaMemcpyAsync vs the
SM-driven accudnn_swap_copy kernel, per-copy time of a burst of back-to-back
copies captured in a CUDA graph (the executor's situation), D2H and H2D,
one direction at a time and both at once on two streams.

  python tools/copy_bench.py [json_out]
"""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1901_06773_b200 import _native  # noqa: E402

lib = _native.cuda_lib()
lib.accudnn_swap_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_ulonglong, ctypes.c_int,
                                  ctypes.c_void_p]
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/copy_bench.json"
BURST = 32
res = []


def run(kind, direction, size, ctas, both=False):
    n = BURST
    dev = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)]
    host = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
    dev2 = [torch.empty(size, dtype=torch.uint8, device="cuda") for _ in range(n)] if both else []
    host2 = [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(n)] if both else []
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def one(dst, src, st):
        if kind == "engine":
            dst.copy_(src, non_blocking=True)
        else:
            rc = lib.accudnn_swap_copy(dst.data_ptr(), src.data_ptr(), size, ctas, st.cuda_stream)
            assert rc == 0, rc

    def body():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        with torch.cuda.stream(s1):
            for i in range(n):
                if direction == "d2h":
                    one(host[i], dev[i], s1)
                else:
                    one(dev[i], host[i], s1)
        if both:
            s2.wait_stream(cur)
            with torch.cuda.stream(s2):
                for i in range(n):
                    one(dev2[i], host2[i], s2)  # the opposite direction (h2d)
            cur.wait_stream(s2)
        cur.wait_stream(s1)

    g = torch.cuda.CUDAGraph()
    body()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        body()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    per = ms * 1e3 / n
    r = {"kind": kind, "dir": "both" if both else direction, "bytes": size, "ctas": ctas,
         "us_per_copy": round(per, 2), "GBps": round(size * n * (2 if both else 1) / (ms * 1e-3) / 1e9, 1)}
    print(json.dumps(r), flush=True)
    res.append(r)


for size in (2048, 131072, 524288, 2 << 20, 8 << 20, 32 << 20):
    for direction in ("d2h", "h2d"):
        run("engine", direction, size, 0)
        for ctas in (4, 8, 16, 32):
            run("kernel", direction, size, ctas)
    run("engine", "d2h", size, 0, both=True)
    run("kernel", "d2h", size, 16, both=True)
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
json.dump(res, open(out, "w"), indent=1)
