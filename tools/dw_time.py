"""dW(fc) GEMM at the C2 shape as bench.py times it (token-major operands, split-K workspace),
50 launches back to back behind a GPU spin, CUDA events: us per launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
d, M = 768, 4096
dev = torch.device("cuda")
ws = torch.empty(2 * 4 * d * d, device=dev)
K.gemm_config(splitk_ws=ws)
dY = torch.randn(M, 4 * d, device=dev)
X = torch.randn(M, d, device=dev)
W = torch.empty(4 * d, d, device=dev)
f = lambda: K.gemm(dY, X, a_mn=True, b_mn=True, C=W)
for _ in range(5):
    f()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
torch.cuda._sleep(300_000_000)
e0.record()
for _ in range(50):
    f()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 50 * 1e3
print(f"dW(fc) {t:.2f} us {2 * M * 4 * d * d / t / 1e6:.0f} TFLOP/s")
