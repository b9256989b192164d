"""ncu target for the bf16 (kind::f16) GEMM: the GPT-2 XL fc shape (16384x6400x1600, one launch) and
the C2 dW(fc) shape (3072x768x4096, token-major operands, the executor's split-K workspace).

ncu --set full --clock-control none -k regex:gemm_tf32 -c 3 python tools/gemm_bf16_ncu.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08633_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
A = torch.randn(16384, 1600, device=dev).to(torch.bfloat16)
B = torch.randn(6400, 1600, device=dev).to(torch.bfloat16)
C = torch.empty(16384, 6400, device=dev)
if len(sys.argv) > 1 and sys.argv[1] == "gelu":  # the fc forward (+ gelu' store) and the GELU' dX GEMM
    bias = torch.randn(6400, device=dev)
    C16 = torch.empty(16384, 6400, device=dev, dtype=torch.bfloat16)
    K.gemm_bf16(A, B, C=C16, c_bf16=True, bias=bias, mode=1, H=C)
    K.gemm_bf16(A, B.t().contiguous(), b_mn=True, C=C16, c_bf16=True, mode=2, H=C)
    torch.cuda.synchronize()
    sys.exit(0)
K.gemm_bf16(A, B, C=C)
d, M = 768, 4096
ws = torch.empty(2 * 4 * d * d, device=dev)
K.gemm_config(splitk_ws=ws)
dY = torch.randn(M, 4 * d, device=dev).to(torch.bfloat16)
X = torch.randn(M, d, device=dev).to(torch.bfloat16)
W = torch.zeros(4 * d, d, device=dev)
K.gemm_bf16(dY, X, a_mn=True, b_mn=True, C=W, beta=1.0)
torch.cuda.synchronize()
