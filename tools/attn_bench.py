"""Fused attention fwd/bwd at the C2 and C3 (XL) shapes, CUDA-event timed with the launches
queued behind a GPU spin (no host gaps; L2 warm)."""
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
    torch.cuda._sleep(100_000_000)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for B, T, H, name in ((8, 512, 12, "C2 gpt2-small b8"), (16, 512, 25, "C3 gpt2-xl b16")):
    qkv = torch.randn(B * T, 3 * H * 64, device=dev)
    dout = torch.randn(B * T, H * 64, device=dev)
    out, lse = K.flash_attention_fwd(qkv, B, T, H)
    fl_fwd = 4.0 * B * H * T * T * 64 / 2  # causal: QK^T + PV over the lower triangle
    t = timeit(lambda: K.flash_attention_fwd(qkv, B, T, H))
    print("%s flash fwd %.1f us  %.0f TFLOP/s (causal-useful)" % (name, t, fl_fwd / t / 1e6))
    t = timeit(lambda: K.flash_attention_bwd(qkv, out, dout, lse, B, T, H))
    print("%s flash bwd %.1f us  %.0f TFLOP/s (causal-useful, 2.5x fwd)" % (name, t, 2.5 * fl_fwd / t / 1e6))
