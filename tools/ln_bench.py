"""LayerNorm fwd / bwd and column sums at the C2 and C3 (XL) shapes: time per launch (queued
behind a GPU spin) and achieved HBM GB/s against the algorithmic bytes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda")


def timeit(f, reps=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda._sleep(50_000_000)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for rows, d in ((4096, 768), (8192, 1600)):
    x = torch.randn(rows, d, device=dev)
    g = torch.randn(d, device=dev)
    b = torch.randn(d, device=dev)
    y, mean, rstd = K.layernorm_fwd(x, g, b)
    t = timeit(lambda: K.layernorm_fwd(x, g, b))
    print(f"ln fwd  {rows}x{d}: {t:7.1f} us  {2 * rows * d * 4 / t / 1e3:7.0f} GB/s")
    dy = torch.randn(rows, d, device=dev)
    dx = torch.zeros(rows, d, device=dev)
    t = timeit(lambda: K.layernorm_bwd(x, g, mean, rstd, dy, dx=dx, accumulate=True))
    print(f"ln bwd  {rows}x{d}: {t:7.1f} us  {4 * rows * d * 4 / t / 1e3:7.0f} GB/s")
    for n in (d, 3 * d, 4 * d):
        dyn = torch.randn(rows, n, device=dev)
        t = timeit(lambda: K.bias_grad(dyn))
        print(f"colsum  {rows}x{n}: {t:7.1f} us  {rows * n * 4 / t / 1e3:7.0f} GB/s")
