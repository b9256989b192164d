"""ncu target for bench.py's roofline kernels: the dW(fc) GEMM exactly as bench.py times it
(token-major operands, the executor's split-K workspace) and the QKV GEMM, at the C2 shapes.

ncu --set full --clock-control none -k regex:gemm_tf32 -c 2 python tools/roofline_ncu.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08633_b200 import kernels as K  # noqa: E402

d, M = 768, 4096
dev = torch.device("cuda")
ws = torch.empty(2 * 4 * d * d, device=dev)
K.gemm_config(splitk_ws=ws)
dY = torch.randn(M, 4 * d, device=dev)
X = torch.randn(M, d, device=dev)
W = torch.empty(4 * d, d, device=dev)
K.gemm(dY, X, a_mn=True, b_mn=True, C=W)
K.gemm_config(splitk_ws=None)
A = torch.randn(M, d, device=dev)
B = torch.randn(3 * d, d, device=dev)
bias = torch.randn(3 * d, device=dev)
C = torch.empty(M, 3 * d, device=dev)
K.gemm(A, B, C=C, bias=bias)
torch.cuda.synchronize()
