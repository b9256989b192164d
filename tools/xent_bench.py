"""softmax-CE over a C2 logits chunk (500 x 50257, row stride 50304), CUDA-event timed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
rows, V, Vp = 500, 50257, 50304
lg = torch.randn(rows, Vp, device="cuda")
tg = torch.randint(0, V, (rows,), device="cuda", dtype=torch.int32)
for _ in range(3): K.softmax_xent(lg, tg, V, 1.0)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20): K.softmax_xent(lg, tg, V, 1.0)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 20 * 1e3
print(f"xent {rows}x{V}: {t:.1f} us, {2 * rows * V * 4 / t / 1e3:.0f} GB/s (1 read + 1 write)")
