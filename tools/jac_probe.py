"""J.sigma / J^T r timing on a cfg2- or cfg4-sized operator through the C ABI (debug).
usage: python tools/jac_probe.py [M] [V]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2507_14046_b200 import _native as N  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 3904
V = int(sys.argv[2]) if len(sys.argv) > 2 else 103296
Vp = (V + 3) // 4 * 4
L = N.lib()
J = torch.randn(M, Vp, device="cuda")
sig = torch.randn(Vp, device="cuda")
rs = torch.randn(M, device="cuda")
g = torch.empty(Vp, device="cuda")
nseg = L.d2ip_jac_nseg(Vp)
part = torch.empty(M * nseg, device="cuda")
wsn = L.d2ip_jac_adj_ws_bytes(M, Vp, 1)
ws = torch.empty(wsn, dtype=torch.uint8, device="cuda")
flush = torch.empty(64 * 1024 * 1024, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)


def t(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts[2:])[len(ts[2:]) // 2]


fwd = lambda: N.check(L.d2ip_jac_fwd(C.c_void_p(J.data_ptr()), 0, C.c_void_p(sig.data_ptr()), 0, M, Vp,  # noqa: E731
                                     C.c_void_p(part.data_ptr()), nseg, 1, st), "fwd")
adj = lambda: N.check(L.d2ip_jac_adj(C.c_void_p(J.data_ptr()), 0, C.c_void_p(rs.data_ptr()), M, Vp,  # noqa: E731
                                     C.c_void_p(g.data_ptr()), 0, C.c_void_p(ws.data_ptr()), wsn, 1, st), "adj")
tf, ta = t(fwd), t(adj)
gb = 4.0 * M * Vp / 1e9
print(f"M={M} Vp={Vp}: jac_fwd {tf:.1f} us ({gb / tf * 1e6 / 1e3:.0f} GB/s)  jac_adj {ta:.1f} us ({gb / ta * 1e6 / 1e3:.0f} GB/s)")
ref = (J.double().T @ rs.double()).float()
print("adj rel err", float((g - ref).norm() / ref.norm()))
