"""Warm CUDA-event timing of single conv layers through the C ABI (debug).

    python tools/conv_bench.py CIN COUT D[xHxW] STRIDE [reps] [precs, e.g. tf32,bf16]

Prints the forward and data-gradient time for precision fp32 (the direct
CUDA-core kernels) and tf32 (the tcgen05 kernels, weight pack included).
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_14046_b200 import _native as N  # noqa: E402

cin, cout, stride = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[4])
dims = [int(v) for v in sys.argv[3].split("x")]
Dd, Hd, Wd = dims if len(dims) == 3 else dims * 3
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
precs = sys.argv[6].split(",") if len(sys.argv) > 6 else ["fp32", "tf32"]
L = N.lib()
Do, Ho, Wo = [(n + stride - 1) // stride for n in (Dd, Hd, Wd)]
x = torch.randn(1, Dd, Hd, Wd, cin, device="cuda")
y = torch.empty(1, Do, Ho, Wo, cout, device="cuda")
gx = torch.empty_like(x)
w = torch.randn(cout * cin * 27 + cout, device="cuda") * 0.05
P = w.numel()
V = Do * Ho * Wo


twins = {}  # bf16 twins (the engine's bf16 layers carry them; TWIN=0 times the fp32-conversion path)
USE_TWIN = os.environ.get("TWIN", "1") == "1"


def act(t, c, dims, prec="fp32"):
    a = N.Act()
    a.ptr, a.c, a.cstride = t.data_ptr(), c, c
    a.d, a.h, a.w = dims
    a.bstride = dims[0] * dims[1] * dims[2] * c
    if prec == "bf16" and USE_TWIN:
        if t.data_ptr() not in twins:
            twins[t.data_ptr()] = t.to(torch.bfloat16)
        a.bf16 = twins[t.data_ptr()].data_ptr()
    return a


st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for prec in precs:
    wsn = max(16, L.d2ip_conv3d_ws_bytes(cin, cout, 3, stride, N.PREC[prec], 1)) + 64 * Dd * Hd * Wd * max(cin, cout) * 4
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")

    def fwd():
        N.check(L.d2ip_conv3d_fwd(act(x, cin, (Dd, Hd, Wd), prec), C.c_void_p(w.data_ptr()),
                                  C.c_void_p(w.data_ptr() + 4 * cout * cin * 27), P, 3, stride,
                                  act(y, cout, (Do, Ho, Wo)), 0,
                                  N.PREC[prec], C.c_void_p(ws.data_ptr()), wsn, 1, st), "fwd")

    def dgrad():
        N.check(L.d2ip_conv3d_dgrad(act(y, cout, (Do, Ho, Wo), prec), C.c_void_p(w.data_ptr()), P, 3, stride,
                                    act(gx, cin, (Dd, Hd, Wd)), 0,
                                    N.PREC[prec], C.c_void_p(ws.data_ptr()), wsn, 1, st), "dgrad")

    gw = torch.zeros(P, device="cuda")
    wgn = max(16, L.d2ip_conv3d_wgrad_ws_bytes(act(x, cin, (Dd, Hd, Wd)), act(y, cout, (Do, Ho, Wo)), 3, 1))
    wgs = torch.empty(wgn, dtype=torch.uint8, device="cuda")

    def wgrad():
        N.check(L.d2ip_conv3d_wgrad(act(x, cin, (Dd, Hd, Wd), prec), act(y, cout, (Do, Ho, Wo), prec), 3, stride,
                                    C.c_void_p(gw.data_ptr()), P, C.c_void_p(wgs.data_ptr()), wgn, N.PREC[prec], 1,
                                    st), "wgrad")

    for name, fn in (("fwd", fwd), ("dgrad", dgrad), ("wgrad", wgrad)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / reps * 1e3
        tf = 2.0 * 27 * cin * cout * V / (us * 1e-6) / 1e12
        print(f"{prec} {name} cin={cin} cout={cout} {Dd}x{Hd}x{Wd} s={stride}: {us:.1f} us, {tf:.1f} TFLOP/s "
              f"({L.d2ip_last_variant().decode()}; weight pack included)")
