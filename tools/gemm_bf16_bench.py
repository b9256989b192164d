"""Time the bf16 (kind::f16) GEMM at the block shapes of C2 (GPT-2 small, M = 4096 tokens) and XL
(b16: M = 16384), next to the TF32 kernel and cuBLAS bf16 (torch.matmul) — CUDA events over 20
back-to-back launches, split-K workspace as in the executor. Prints one JSON line (TFLOP/s)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {  # name: (M, N, K, a_mn, b_mn)
    "qkv": (4096, 2304, 768, 0, 0), "o": (4096, 768, 768, 0, 0), "fc": (4096, 3072, 768, 0, 0),
    "pr": (4096, 768, 3072, 0, 0), "dX(pr)": (4096, 3072, 768, 0, 1), "dX(fc)": (4096, 768, 3072, 0, 1),
    "dW(pr)": (768, 3072, 4096, 1, 1), "dW(fc)": (3072, 768, 4096, 1, 1), "dW(qkv)": (2304, 768, 4096, 1, 1),
    "xl fc": (16384, 6400, 1600, 0, 0), "xl pr": (16384, 1600, 6400, 0, 0), "xl dX(pr)": (16384, 6400, 1600, 0, 1),
    "xl dW(fc)": (6400, 1600, 16384, 1, 1), "sq 8192": (8192, 8192, 8192, 0, 0),
}


def timeit(f, reps=20):
    import torch
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def main():
    import torch
    from paper_2110_08633_b200 import kernels as K
    dev = torch.device("cuda")
    ws = torch.empty(2 * 6400 * 1600 + 16, device=dev)
    K.gemm_config(splitk_ws=ws)
    out = {}
    for name, (M, N, Kd, amn, bmn) in SHAPES.items():
        A = torch.randn(Kd, M, device=dev) if amn else torch.randn(M, Kd, device=dev)
        B = torch.randn(Kd, N, device=dev) if bmn else torch.randn(N, Kd, device=dev)
        A16, B16 = A.to(torch.bfloat16), B.to(torch.bfloat16)
        C = torch.zeros(M, N, device=dev)
        beta = 1.0 if name.startswith("dW") or "dW" in name else 0.0
        t16 = timeit(lambda: K.gemm_bf16(A16, B16, a_mn=bool(amn), b_mn=bool(bmn), C=C, beta=beta))
        t32 = timeit(lambda: K.gemm(A, B, a_mn=bool(amn), b_mn=bool(bmn), M=M, N=N, K=Kd, C=C, beta=beta))
        Am = A16.t() if amn else A16
        Bm = B16 if bmn else B16.t()
        C16 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        tcb = timeit(lambda: torch.matmul(Am, Bm, out=C16))
        fl = 2.0 * M * N * Kd
        out[name] = {"bf16": round(fl / t16 / 1e12, 1), "tf32": round(fl / t32 / 1e12, 1),
                     "cublas_bf16": round(fl / tcb / 1e12, 1), "bf16_us": round(t16 * 1e6, 2)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
