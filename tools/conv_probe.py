"""Run one tcgen05 conv layer through the C ABI (for ncu captures).
usage: python tools/conv_probe.py CIN COUT D [reps] [dgrad]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_14046_b200 import _native as N  # noqa: E402

cin, cout, D = (int(a) for a in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
L = N.lib()
x = torch.randn(1, D, D, D, cin, device="cuda")
y = torch.empty(1, D, D, D, cout, device="cuda")
w = torch.randn(cout * cin * 27 + cout, device="cuda") * 0.05


def act(t, c):
    a = N.Act()
    a.ptr, a.d, a.h, a.w, a.c, a.cstride = t.data_ptr(), D, D, D, c, c
    a.bstride = D * D * D * c
    return a


wsn = L.d2ip_conv3d_ws_bytes(cin, cout, 3, 1, N.PREC["tf32"], 1)
ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(reps):
    N.check(L.d2ip_conv3d_fwd(act(x, cin), C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr() + 4 * cout * cin * 27),
                              0, 3, 1, act(y, cout), 0, N.PREC["tf32"], C.c_void_p(ws.data_ptr()), wsn, 1, st), "conv")
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    L.d2ip_conv3d_fwd(act(x, cin), C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr() + 4 * cout * cin * 27),
                      0, 3, 1, act(y, cout), 0, N.PREC["tf32"], C.c_void_p(ws.data_ptr()), wsn, 1, st)
e.record()
torch.cuda.synchronize()
t = s.elapsed_time(e) / 20 * 1e-3
print(f"conv {cin}->{cout} @{D}^3: {t*1e6:.1f} us (incl. pack), {2*27*cin*cout*D**3/t/1e12:.2f} TFLOP/s")
