"""ncu target for bench.py's bf16 roofline entries: the bf16 GEMM at the C2 fc shape (4096x3072x768)
and at GPT-2 XL's fc shape (16384x6400x1600), plain fp32 store, as bench.py times them.

ncu --set full --clock-control none -k regex:gemm_tf32 -c 2 python tools/roofline_bf16_ncu.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08633_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
for M, N, Kd in ((4096, 3072, 768), (16384, 6400, 1600)):
    A = torch.randn(M, Kd, device=dev).to(torch.bfloat16)
    B = torch.randn(N, Kd, device=dev).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev)
    K.gemm_bf16(A, B, C=C)
torch.cuda.synchronize()
