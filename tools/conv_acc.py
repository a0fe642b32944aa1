"""Op-level accuracy of the tensor-core convolutions vs a float64 reference (debug).
usage: python tools/conv_acc.py PREC "cin cout DxHxW stride" ...   (prints fwd / dgrad / wgrad rel errors)"""
import ctypes as C
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
from paper_2507_14046_b200 import _native as N  # noqa: E402

L = N.lib()
prec = sys.argv[1]
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def act(t, c, dims):
    a = N.Act()
    a.ptr, a.c, a.cstride = t.data_ptr(), c, c
    a.d, a.h, a.w = dims
    a.bstride = dims[0] * dims[1] * dims[2] * c
    if prec == "bf16":
        tw = t.to(torch.bfloat16)
        act.keep.append(tw)
        a.bf16 = tw.data_ptr()
    return a


act.keep = []


def rel(a, b):
    d = (a.double() - b)
    return float(d.norm() / b.norm()), float(d.abs().max() / b.abs().max())


for spec in sys.argv[2:]:
    cin, cout, dims, stride = spec.split()
    cin, cout, stride = int(cin), int(cout), int(stride)
    D, H, W = (int(v) for v in dims.split("x"))
    Do, Ho, Wo = [(n + stride - 1) // stride for n in (D, H, W)]
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(1, D, H, W, cin, device="cuda", generator=g)
    gy = torch.randn(1, Do, Ho, Wo, cout, device="cuda", generator=g)
    w = torch.randn(cout * cin * 27 + cout, device="cuda", generator=g) * (2.0 / (27 * cin)) ** 0.5
    P = w.numel()
    wt = w[:cout * cin * 27].view(cout, cin, 3, 3, 3).double()
    bias = w[cout * cin * 27:].double()
    x64 = x.double().permute(0, 4, 1, 2, 3).requires_grad_(True)
    wt64 = wt.clone().requires_grad_(True)
    y64 = F.conv3d(x64, wt64, bias, stride=stride, padding=1)
    y64.backward(gy.double().permute(0, 4, 1, 2, 3))
    y = torch.empty(1, Do, Ho, Wo, cout, device="cuda")
    gx = torch.empty_like(x)
    gw = torch.zeros(P, device="cuda")
    wsn = max(16, L.d2ip_conv3d_ws_bytes(cin, cout, 3, stride, N.PREC[prec], 1)) + 64 * D * H * W * max(cin, cout) * 4
    ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
    N.check(L.d2ip_conv3d_fwd(act(x, cin, (D, H, W)), C.c_void_p(w.data_ptr()),
                              C.c_void_p(w.data_ptr() + 4 * cout * cin * 27), P, 3, stride, act(y, cout, (Do, Ho, Wo)),
                              0, N.PREC[prec], C.c_void_p(ws.data_ptr()), wsn, 1, st), "fwd")
    vf = L.d2ip_last_variant().decode()
    N.check(L.d2ip_conv3d_dgrad(act(gy, cout, (Do, Ho, Wo)), C.c_void_p(w.data_ptr()), P, 3, stride,
                                act(gx, cin, (D, H, W)), 0, N.PREC[prec], C.c_void_p(ws.data_ptr()), wsn, 1, st),
            "dgrad")
    vd = L.d2ip_last_variant().decode()
    wgn = max(16, L.d2ip_conv3d_wgrad_ws_bytes(act(x, cin, (D, H, W)), act(gy, cout, (Do, Ho, Wo)), 3, stride))
    wgs = torch.empty(wgn, dtype=torch.uint8, device="cuda")
    N.check(L.d2ip_conv3d_wgrad(act(x, cin, (D, H, W)), act(gy, cout, (Do, Ho, Wo)), 3, stride,
                                C.c_void_p(gw.data_ptr()), P, C.c_void_p(wgs.data_ptr()), wgn, N.PREC[prec], 1, st),
            "wgrad")
    vw = L.d2ip_last_variant().decode()
    torch.cuda.synchronize()
    ef = rel(y.permute(0, 4, 1, 2, 3), y64.detach())
    ed = rel(gx.permute(0, 4, 1, 2, 3), x64.grad)
    ew = rel(gw[:cout * cin * 27].view(cout, cin, 3, 3, 3), wt64.grad)
    print(f"{prec} {cin}->{cout} {dims} s{stride}: fwd {ef[0]:.2e}/{ef[1]:.2e} [{vf}]  dgrad {ed[0]:.2e}/{ed[1]:.2e} "
          f"[{vd}]  wgrad {ew[0]:.2e}/{ew[1]:.2e} [{vw}]")
