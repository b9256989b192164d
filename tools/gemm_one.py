"""One workload GEMM shape, timed without host overhead: 20 launches queued behind a GPU spin
(torch.cuda._sleep) and bracketed by CUDA events (the executor enqueues ahead of the GPU, so
host launch cost is hidden there too). Also the target of single-kernel ncu captures.

python tools/gemm_one.py [shape ...]     (names from tools/gemm_bench.SHAPES; default: all)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08633_b200 import kernels as K  # noqa: E402
from tools.gemm_bench import SHAPES  # noqa: E402

names = sys.argv[1:] or list(SHAPES)
dev = torch.device("cuda")
out = {}
for name in names:
    M, N, Kd, amn, bmn = SHAPES[name]
    A = torch.randn(Kd, M, device=dev) if amn else torch.randn(M, Kd, device=dev)
    if name == "logits":
        B = torch.randn(N, Kd, device=dev)
        C = torch.empty(M, 50304, device=dev)
    else:
        B = torch.randn(Kd, N, device=dev) if bmn else torch.randn(N, Kd, device=dev)
        C = torch.empty(M, N, device=dev)
    f = lambda: K.gemm(A, B, a_mn=bool(amn), b_mn=bool(bmn), M=M, N=N, K=Kd, C=C, ldc=C.stride(0))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    # the GPU spins while the host queues the timed launches, so the events bracket
    # back-to-back kernels with no host launch gaps
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000_000)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 / 1e3
    out[name] = {"us": round(t * 1e6, 2), "tflops": round(2.0 * M * N * Kd / t / 1e12, 1)}
print(json.dumps(out))
