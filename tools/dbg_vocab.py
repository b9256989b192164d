import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda")
torch.manual_seed(0)
for rows, d, V, ldc in ((256, 128, 50257, 50304), (256, 128, 4096, 4096), (512, 128, 50257, 50304), (256, 768, 50257, 50304)):
    z = torch.randn(rows, d, device=dev)
    wte = torch.randn(V, d, device=dev) * 0.02
    logits = torch.zeros(rows, ldc, device=dev)
    K.gemm(z, wte, C=logits, M=rows, N=V, K=d, ldc=ldc)
    ref = z @ wte.T
    err = (logits[:, :V] - ref).abs()
    bad = (err > 1e-2).nonzero()
    print(rows, d, V, "bad", bad.shape[0], "of", rows * V)
    if bad.shape[0]:
        cols = bad[:, 1]
        print("  col tiles (256) bad:", sorted(set((cols // 256).tolist()))[:20], "... rows:", sorted(set((bad[:, 0] // 32).tolist())))
        print("  col within tile:", sorted(set((cols % 256 // 32).tolist())))
