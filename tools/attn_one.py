"""One fused-attention fwd + bwd at the C2 shape (ncu capture target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda")
B, T, H = 8, 512, 12
qkv = torch.randn(B * T, 3 * H * 64, device=dev)
dout = torch.randn(B * T, H * 64, device=dev)
for _ in range(3):
    out, lse = K.flash_attention_fwd(qkv, B, T, H)
    K.flash_attention_bwd(qkv, out, dout, lse, B, T, H)
torch.cuda.synchronize()
