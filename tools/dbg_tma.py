import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
l = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "dbg_tma.so"))
l.dbg_tma.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_long, ctypes.c_long, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
src = torch.arange(32 * 128, dtype=torch.float32, device="cuda").view(32, 128)  # [K=32 rows][M=128]
out = torch.zeros(1024, device="cuda")
rc = l.dbg_tma(src.data_ptr(), 128, 32, 128, out.data_ptr(), 32, 0)
print("rc", rc)
t = out.view(32, 32)
print(t[:3, :12].tolist())
print("row1", t[1].tolist())
