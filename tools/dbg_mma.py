import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
l = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "dbg_tma.so"))
l.dbg_mma.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, ctypes.c_int, ctypes.c_int, ctypes.c_int]
torch.manual_seed(0)
A = torch.randn(128, 32, device="cuda")   # [M][K]
B = torch.randn(128, 32, device="cuda")   # [N][K]
A_mn = A.T.contiguous()                    # [K][M]
ref = A[:, :8] @ B[:, :8].T               # one MMA, K=8
def idesc(M, N, amn, bmn):
    return (1 << 4) | (2 << 7) | (2 << 10) | (amn << 15) | (bmn << 16) | ((N >> 3) << 17) | ((M >> 4) << 24)
out = torch.zeros(128 * 128, device="cuda")
ref16 = A[:, :8] @ B[:, :8].T
for name, stride, lbo, sbo, ltype, swz in [("b32_l4096_s512", 4096, 4096, 512, 1, 4), ("b32_l512_s4096", 4096, 512, 4096, 1, 4),
        ("b32_l4096_s1024", 4096, 4096, 1024, 1, 4), ("sw128std", 4096, 4096, 1024, 2, 3)]:
    out.zero_()
    rc = l.dbg_mma(A_mn.data_ptr(), B.data_ptr(), out.data_ptr(), stride, lbo, sbo, idesc(128, 128, 1, 0), 0, ltype, swz)
    o = out.view(128, 128)
    print(name, "rc", rc, "rel", ((o - ref).norm() / ref.norm()).item(), "absmax", o.abs().max().item())
