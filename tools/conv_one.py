"""One conv layer forward (or dgrad) through the C ABI, for ncu (debug).
usage: python tools/conv_one.py CIN COUT DxHxW [fwd|dgrad] [reps] [prec]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_14046_b200 import _native as N  # noqa: E402

cin, cout = int(sys.argv[1]), int(sys.argv[2])
D, H, W = (int(v) for v in sys.argv[3].split("x"))
which = sys.argv[4] if len(sys.argv) > 4 else "fwd"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
prec = sys.argv[6] if len(sys.argv) > 6 else "tf32"
L = N.lib()
x = torch.randn(1, D, H, W, cin, device="cuda")
y = torch.randn(1, D, H, W, cout, device="cuda")
w = torch.randn(cout * cin * 27 + cout, device="cuda") * 0.05


def act(t, c):
    a = N.Act()
    a.ptr, a.d, a.h, a.w, a.c, a.cstride = t.data_ptr(), D, H, W, c, c
    a.bstride = D * H * W * c
    return a


wsn = max(16, L.d2ip_conv3d_ws_bytes(cin, cout, 3, 1, N.PREC[prec], 1)) + 64 * D * H * W * max(cin, cout) * 4
ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(reps):
    if which == "fwd":
        N.check(L.d2ip_conv3d_fwd(act(x, cin), C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr() + 4 * cout * cin * 27),
                                  0, 3, 1, act(y, cout), 0, N.PREC[prec], C.c_void_p(ws.data_ptr()), wsn, 1, st), "fwd")
    else:
        N.check(L.d2ip_conv3d_dgrad(act(y, cout), C.c_void_p(w.data_ptr()), 0, 3, 1, act(x, cin), 0, N.PREC[prec],
                                    C.c_void_p(ws.data_ptr()), wsn, 1, st), "dgrad")
torch.cuda.synchronize()
print(L.d2ip_last_variant().decode())
