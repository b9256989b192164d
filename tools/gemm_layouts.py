"""The weight-gradient shape (M=3072, N=768, K=4096) under all four operand layouts: isolates the
cost of MN-major (transposed) smem operands from the shape itself. CUDA events around 20 launches
queued behind a GPU spin."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_08633_b200 import kernels as K  # noqa: E402

M, N, Kd = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (3072, 768, 4096)))
dev = torch.device("cuda")
ws = torch.empty(32 << 20, device=dev)  # split-K partials (used when the dispatcher splits)
K.gemm_config(False, ws)
out = {}
for amn in (0, 1):
    for bmn in (0, 1):
        A = torch.randn(Kd, M, device=dev) if amn else torch.randn(M, Kd, device=dev)
        B = torch.randn(Kd, N, device=dev) if bmn else torch.randn(N, Kd, device=dev)
        C = torch.empty(M, N, device=dev)
        f = lambda: K.gemm(A, B, a_mn=bool(amn), b_mn=bool(bmn), M=M, N=N, K=Kd, C=C, ldc=C.stride(0))
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000_000)
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        out[f"a_mn={amn} b_mn={bmn}"] = {"us": round(us, 2), "tflops": round(2 * M * N * Kd / us / 1e6, 1)}
print(json.dumps({"shape": [M, N, Kd], **out}))
