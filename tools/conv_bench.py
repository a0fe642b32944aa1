"""Warm CUDA-event timing of single conv layers through the C ABI (debug).

    python tools/conv_bench.py CIN COUT D STRIDE [reps]

Prints the forward and data-gradient time for precision fp32 (the direct
CUDA-core kernels) and tf32 (the tcgen05 kernels, weight pack included).
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_14046_b200 import _native as N  # noqa: E402

cin, cout, D, stride = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 50
L = N.lib()
Do = (D + stride - 1) // stride
x = torch.randn(1, D, D, D, cin, device="cuda")
y = torch.empty(1, Do, Do, Do, cout, device="cuda")
gx = torch.empty_like(x)
w = torch.randn(cout * cin * 27 + cout, device="cuda") * 0.05
P = w.numel()


def act(t, c, d):
    a = N.Act()
    a.ptr, a.d, a.h, a.w, a.c, a.cstride = t.data_ptr(), d, d, d, c, c
    a.bstride = d * d * d * c
    return a


st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for prec in ("fp32", "tf32"):
    wsn = max(16, L.d2ip_conv3d_ws_bytes(cin, cout, 3, stride, N.PREC[prec], 1)) + 64 * D ** 3 * max(cin, cout) * 4
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")

    def fwd():
        N.check(L.d2ip_conv3d_fwd(act(x, cin, D), C.c_void_p(w.data_ptr()),
                                  C.c_void_p(w.data_ptr() + 4 * cout * cin * 27), P, 3, stride, act(y, cout, Do), 0,
                                  N.PREC[prec], C.c_void_p(ws.data_ptr()), wsn, 1, st), "fwd")

    def dgrad():
        N.check(L.d2ip_conv3d_dgrad(act(y, cout, Do), C.c_void_p(w.data_ptr()), P, 3, stride, act(gx, cin, D), 0,
                                    N.PREC[prec], C.c_void_p(ws.data_ptr()), wsn, 1, st), "dgrad")

    for name, fn in (("fwd", fwd), ("dgrad", dgrad)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(f"{prec} {name} cin={cin} cout={cout} D={D} s={stride}: {a.elapsed_time(b) / reps * 1e3:.1f} us "
              f"({L.d2ip_last_variant().decode()})")
