"""GEMM epilogue cost at the C2 MLP shape: plain / bias / bias+residual / GELU / GELU'."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda")
M, N, Kd = 4096, 3072, 768
A = torch.randn(M, Kd, device=dev); B = torch.randn(N, Kd, device=dev) * 0.05
C = torch.empty(M, N, device=dev); H = torch.empty(M, N, device=dev); R = torch.randn(M, N, device=dev)
bias = torch.randn(N, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
cases = {"plain": dict(), "bias": dict(bias=bias), "bias+R": dict(bias=bias, R=R), "gelu": dict(bias=bias, mode=1, H=H),
         "gelu_bwd": dict(mode=2, H=R)}
for name, kw in cases.items():
    f = lambda: K.gemm(A, B, C=C, **kw)
    for _ in range(3): f()
    ts = []
    for _ in range(10):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"{name:9s} median {ts[5]:7.1f} us  {2*M*N*Kd/ts[5]/1e6:6.1f} TF/s (L2 flushed)")
