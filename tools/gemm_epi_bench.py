"""GEMMs with their executor epilogues at the XL (C3) shapes, queued behind a GPU spin:
fc + GELU (writes pre-activation too), dact = dY W (x) GELU'(H), mlp_proj + residual, dW with
beta = 1 accumulation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda")
M, d = 8192, 1600


def timeit(f, reps=10):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda._sleep(100_000_000)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


x = torch.randn(M, d, device=dev)
w_fc = torch.randn(4 * d, d, device=dev) * 0.02
b_fc = torch.randn(4 * d, device=dev)
act = torch.empty(M, 4 * d, device=dev)
pre = torch.empty(M, 4 * d, device=dev)
fl = 2.0 * M * 4 * d * d
t = timeit(lambda: K.gemm(x, w_fc, C=act, bias=b_fc, mode=1, H=pre))
print(f"fc+gelu   {t:7.1f} us {fl / t / 1e6:6.0f} TFLOP/s")
dh = torch.randn(M, d, device=dev)
w_pr = torch.randn(d, 4 * d, device=dev) * 0.02  # [d, 4d]: B for dY W is MN-major
dact = torch.empty(M, 4 * d, device=dev)
t = timeit(lambda: K.gemm(dh, w_pr, b_mn=True, M=M, N=4 * d, K=d, C=dact, mode=2, H=pre))
print(f"dact      {t:7.1f} us {fl / t / 1e6:6.0f} TFLOP/s")
out = torch.empty(M, d, device=dev)
b_pr = torch.randn(d, device=dev)
t = timeit(lambda: K.gemm(act, w_pr, C=out, bias=b_pr, R=x))
print(f"proj+res  {t:7.1f} us {fl / t / 1e6:6.0f} TFLOP/s")
gw = torch.zeros(4 * d, d, device=dev)
t = timeit(lambda: K.gemm(dact, x, a_mn=True, b_mn=True, M=4 * d, N=d, K=M, C=gw, beta=1.0))
print(f"dW(fc)    {t:7.1f} us {fl / t / 1e6:6.0f} TFLOP/s")
