"""Debug harness for the tcgen05 wgrad: one case, prints partial stats."""
import ctypes as C
import sys
import torch
import torch.nn.functional as F
sys.path.insert(0, ".")
from paper_2507_14046_b200 import _native as N

def act_of(t, c=None, coff=0):
    B, D, H, W, CS = t.shape
    a = N.Act(); a.ptr = t.data_ptr() + coff * 4; a.d, a.h, a.w = D, H, W
    a.c = CS if c is None else c; a.cstride = CS; a.bstride = D * H * W * CS
    return a

cin, cout, ks, sp = [int(v) for v in sys.argv[1:4]] + [tuple(int(v) for v in sys.argv[4].split(","))]
torch.manual_seed(1)
B = 1
x = torch.randn(B, cin, *sp)
gy = torch.randn(B, cout, *sp)
w = torch.zeros(cout, cin, ks, ks, ks, requires_grad=True)
bb = torch.zeros(cout, requires_grad=True)
y = F.conv3d(x, w, bb, padding=ks // 2); y.backward(gy)
xd = x.permute(0, 2, 3, 4, 1).contiguous().cuda(); gyd = gy.permute(0, 2, 3, 4, 1).contiguous().cuda()
P = cout * cin * ks ** 3 + cout
gw = torch.zeros(B, P, device="cuda")
L = N.lib()
n = L.d2ip_conv3d_wgrad_ws_bytes(act_of(xd), act_of(gyd), ks, B)
ws = torch.full((n // 4 + 4,), -777.0, device="cuda")
rc = L.d2ip_conv3d_wgrad(act_of(xd), act_of(gyd), ks, 1, C.c_void_p(gw.data_ptr()), P, C.c_void_p(ws.data_ptr()), n,
                         1, B, C.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("rc", rc, L.d2ip_last_variant(), L.d2ip_last_error())
nW = cout * cin * ks ** 3
ref = w.grad.reshape(-1)
got = gw[0, :nW].cpu()
print("ref norm", ref.norm().item(), "got norm", got.norm().item(), "rel", ((got - ref).norm() / ref.norm()).item())
print("bias ref", bb.grad[:4].tolist(), "got", gw[0, nW:nW + 4].tolist())
print("ws stats: n", ws.numel(), "sentinel left", (ws == -777.0).sum().item(), "zeros", (ws == 0).sum().item(),
      "absmax", ws[ws != -777.0].abs().max().item() if (ws != -777.0).any() else None)
# per-tap compare (t, ci, co)
refT = w.grad.permute(2, 3, 4, 1, 0).reshape(ks ** 3, cin, cout)
gotT = got.reshape(cout, cin, ks ** 3).permute(2, 1, 0)
for t in range(min(ks ** 3, 27)):
    e = ((gotT[t] - refT[t]).norm() / refT[t].norm()).item()
    print("tap", t, "rel", round(e, 6), "got00", round(gotT[t][0, 0].item(), 4), "ref00", round(refT[t][0, 0].item(), 4))
