"""In-stream time and achieved HBM GB/s of the HBM-bound shard kernels at the C2 (4096 x 768) and
XL b16 (8192 x 1600) shapes: CUDA events; before each launch L2 is flushed by READING a 512 MB
buffer (a write flush leaves ~126 MB of dirty lines that the timed kernel would pay to evict).
A same-bytes device copy (torch clone) is timed the same way as the practical bound."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda")
flush = torch.ones(128 << 20, dtype=torch.float32, device=dev)
sink = torch.empty(1, device=dev)


def t(f, reps=10, cold=True):
    f()
    ts = []
    for _ in range(reps):
        if cold:
            sink.copy_(flush.sum())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for rows, d in ((4096, 768), (8192, 1600)):
    x = torch.randn(rows, d, device=dev); g = torch.randn(d, device=dev); b = torch.randn(d, device=dev)
    dy = torch.randn(rows, d, device=dev); dx = torch.zeros(rows, d, device=dev)
    dyf = torch.randn(rows, 4 * d, device=dev)
    y, mean, rstd = K.layernorm_fwd(x, g, b)
    cases = [("ln_fwd", lambda: K.layernorm_fwd(x, g, b), 2 * rows * d * 4),
             ("ln_bwd (dx + dg/db)", lambda: K.layernorm_bwd(x, g, mean, rstd, dy, dx=dx, accumulate=True),
              (4 * rows * d + 2 * rows * d) * 4),
             ("bias_grad 4d", lambda: K.bias_grad(dyf), rows * 4 * d * 4)]
    big = torch.randn(rows * d * 3, device=dev)
    cases.append(("copy (same bytes as ln_bwd)", lambda: big.clone(), 6 * rows * d * 4))
    cases.append(("copy (same bytes as ln_fwd)", lambda: x.clone(), 2 * rows * d * 4))
    for name, f, byts in cases:
        us, wus = t(f), t(f, cold=False)
        print(f"{rows}x{d} {name:28s} cold {us:7.1f} us {byts / us / 1e3:6.0f} GB/s | warm {wus:7.1f} us")
