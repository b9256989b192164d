"""Attention fwd/bwd pieces at the C2 shape, CUDA-event timed (standalone, L2 warm)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08633_b200 import kernels as K
dev = torch.device("cuda")
B, T, H = 8, 512, 12
qkv = torch.randn(B * T, 3 * H * 64, device=dev)
dout = torch.randn(B * T, H * 64, device=dev)
Md = B * T * H * 64
def timeit(f, reps=20):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
for wf_mult, name in ((8, "fwd work=8Md (C2 runner)"), (32, "fwd work=32Md")):
    print(name, "%.1f us" % timeit(lambda: K.attention_fwd(qkv, B, T, H, work_floats=wf_mult * Md)))
for wf_mult, name in ((5, "bwd work=5Md (C2 runner)"), (9, "bwd work=9Md"), (16, "bwd work=16Md (1 chunk)")):
    print(name, "%.1f us" % timeit(lambda: K.attention_bwd(qkv, dout, B, T, H, work_floats=wf_mult * Md)))
out, lse = K.flash_attention_fwd(qkv, B, T, H)
fl_fwd = 4.0 * B * H * T * T * 64 / 2  # causal: QK^T + PV over the lower triangle
t = timeit(lambda: K.flash_attention_fwd(qkv, B, T, H))
print("flash fwd %.1f us  %.0f TFLOP/s (causal-useful)" % (t, fl_fwd / t / 1e6))
t = timeit(lambda: K.flash_attention_bwd(qkv, out, dout, lse, B, T, H))
print("flash bwd %.1f us  %.0f TFLOP/s (causal-useful, 2.5x fwd)" % (t, 2.5 * fl_fwd / t / 1e6))
