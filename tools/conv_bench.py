"""Times the tcgen05 conv kernels on every distinct ResNet-152 conv shape at
k images (default 27 = the tuner's k* at 8 GiB) next to cuDNN TF32 (torch,
channels_last) as a yardstick.  Usage: conv_bench.py [k] [json_out] [mode]
mode: table (the committed tuned table, default) | retune (autotune every
shape, candidates include stream-K; the table is written next to json_out)
| sk (stream-K forced on every launch)"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1901_06773_b200 import _native, trainer  # noqa: E402


def shapes(k):
    _, d = trainer.export_network("resnet152", 224, 1000)
    ops = d["ops"]
    seen = {}
    for o in ops:
        if o["kind"] != "conv":
            continue
        src = ops[o["in0"]]["out"] if o["in0"] >= 0 else [224, 224, 4]
        key = (k, o["cin"] if o["in0"] >= 0 else 4, src[0], src[1], o["cout"], o["r"], o["stride"], o["pad"])
        seen[key] = seen.get(key, 0) + 1
    return seen


def timeit(fn, iters=20, graph=False):
    """device time per call; graph=True replays `iters` calls captured in a
    CUDA graph (no host launch/encode cost, as inside the training step)"""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(iters):
                    fn(s)
            g.replay()
            torch.cuda.synchronize()
            a.record(s)
            g.replay()
            b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / iters
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    lib = _native.cuda_lib()
    import os
    tune = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "b200",
                        "conv_tune.txt")
    mode_arg = sys.argv[3] if len(sys.argv) > 3 else "table"
    if mode_arg == "table" and os.path.exists(tune):
        _native.conv_tune_import(open(tune).read())
    if mode_arg == "retune":
        lib.accudnn_conv_autotune(1)
    if mode_arg == "sk":
        lib.accudnn_conv_force_cfg(0, -1, 0)
    dev = torch.device("cuda:0")
    torch.backends.cudnn.allow_tf32 = True
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.benchmark = True
    out = []
    tot = {"ours": 0.0, "cudnn": 0.0, "gflop": 0.0}
    for (n, c, h, w, kk, r, st, pad), count in shapes(k).items():
        p = (h + 2 * pad - r) // st + 1
        q = (w + 2 * pad - r) // st + 1
        d = _native.ConvDesc(n, h, w, c, kk, r, r, st, pad, p, q)
        x = torch.randn(n, h, w, c, device=dev)
        wt = torch.randn(kk, r, r, c, device=dev) * 0.01
        y = torch.empty(n, p, q, kk, device=dev)
        dy = torch.randn(n, p, q, kk, device=dev)
        dx = torch.empty_like(x)
        dw = torch.empty_like(wt)
        flops = 2.0 * n * p * q * kk * c * r * r
        # cuDNN yardstick (NCHW logical view of the NHWC buffers = channels_last)
        xc = x.permute(0, 3, 1, 2)
        wc = wt.permute(0, 3, 1, 2)
        dyc = dy.permute(0, 3, 1, 2)
        res = {"shape": f"{h}x{w} {c}->{kk} r{r} s{st}", "count": count}
        S = lambda s: ctypes.c_void_p(s.cuda_stream) if s is not None else None  # noqa: E731
        for mode, fn, cfn in (
            ("fwd", lambda s=None: lib.accudnn_conv_fwd(ctypes.byref(d), x.data_ptr(), wt.data_ptr(), y.data_ptr(), 0, S(s)),
             lambda s=None: torch.nn.functional.conv2d(xc, wc, stride=st, padding=pad)),
            ("dgrad", lambda s=None: lib.accudnn_conv_dgrad(ctypes.byref(d), dy.data_ptr(), wt.data_ptr(), dx.data_ptr(), 0, S(s)),
             lambda s=None: torch.ops.aten.convolution_backward(dyc, xc, wc, None, [st, st], [pad, pad], [1, 1], False, [0, 0], 1, [True, False, False])),
            ("wgrad", lambda s=None: lib.accudnn_conv_wgrad(ctypes.byref(d), x.data_ptr(), dy.data_ptr(), dw.data_ptr(), 0, 0, S(s)),
             lambda s=None: torch.ops.aten.convolution_backward(dyc, xc, wc, None, [st, st], [pad, pad], [1, 1], False, [0, 0], 1, [False, True, False]))):
            if mode == "dgrad" and x.shape[-1] == 4:
                continue
            ms = timeit(fn, graph=True)
            cms = timeit(cfn, graph=True)
            res[mode] = {"ms": round(ms, 4), "tflops": round(flops / ms / 1e9, 1),
                         "cudnn_ms": round(cms, 4), "cudnn_tflops": round(flops / cms / 1e9, 1)}
            tot["ours"] += ms * count
            tot["cudnn"] += cms * count
            tot["gflop"] += flops * count / 1e9
        out.append(res)
        print(json.dumps(res), flush=True)
    tot["ours_tflops"] = round(tot["gflop"] / tot["ours"], 1)
    tot["cudnn_tflops"] = round(tot["gflop"] / tot["cudnn"], 1)
    print("TOTAL", json.dumps(tot), flush=True)
    if len(sys.argv) > 2:
        json.dump({"k": k, "shapes": out, "total": tot}, open(sys.argv[2], "w"), indent=1)
        if mode_arg == "retune":
            with open(sys.argv[2].rsplit(".", 1)[0] + "_tune.txt", "w") as f:
                f.write(_native.conv_tune_export())


if __name__ == "__main__":
    main()
