"""ncu target: the C2 fc-shape GEMM (4096x3072x768) with a plain fp32 store, TF32 and bf16 operands.

ncu --set full --import-source on -k regex:gemm_tf32 -c 2 python tools/gemm_c2_ncu.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08633_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda")
A = torch.randn(4096, 768, device=dev)
B = torch.randn(3072, 768, device=dev)
C = torch.empty(4096, 3072, device=dev)
K.gemm(A, B, C=C)
K.gemm_bf16(A.to(torch.bfloat16), B.to(torch.bfloat16), C=C)
torch.cuda.synchronize()
