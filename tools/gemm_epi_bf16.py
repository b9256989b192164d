"""bf16 GEMM epilogue cost at the block shapes (CUDA events, 20 back-to-back launches): plain fp32
store, bf16 store, GELU with a bf16 activation (forward task), GELU + fp32 pre-activation (backward
recompute), GELU' with a bf16 output. Prints one JSON line of microseconds per launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


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
    return round(e0.elapsed_time(e1) / reps * 1e3, 2)


def main():
    import torch
    from paper_2110_08633_b200 import kernels as K
    dev = torch.device("cuda")
    out = {}
    for name, (M, N, Kd) in {"c2 fc": (4096, 3072, 768), "xl fc": (16384, 6400, 1600)}.items():
        A = torch.randn(M, Kd, device=dev).to(torch.bfloat16)
        B = (torch.randn(N, Kd, device=dev) * 0.05).to(torch.bfloat16)
        bias = torch.randn(N, device=dev)
        C = torch.empty(M, N, device=dev)
        C16 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        H = torch.empty(M, N, device=dev)
        Bt = B.t().contiguous()  # [K][N]: dX-style B MN-major operand of the same GEMM
        r = {
            "store_f32": timeit(lambda: K.gemm_bf16(A, B, C=C)),
            "store_bf16": timeit(lambda: K.gemm_bf16(A, B, C=C16, c_bf16=True)),
            "bias_store_f32": timeit(lambda: K.gemm_bf16(A, B, C=C, bias=bias)),
            "gelu_bf16": timeit(lambda: K.gemm_bf16(A, B, C=C16, c_bf16=True, bias=bias, mode=1)),
            "gelu_bf16_hout_f32": timeit(lambda: K.gemm_bf16(A, B, C=C16, c_bf16=True, bias=bias, mode=1, H=H)),
            "gelu_bwd_bf16": timeit(lambda: K.gemm_bf16(A, Bt, b_mn=True, C=C16, c_bf16=True, mode=2, H=H)),
            "store_f32_bmn": timeit(lambda: K.gemm_bf16(A, Bt, b_mn=True, C=C)),
        }
        r["mma_only_us_at_1.4PF"] = round(2.0 * M * N * Kd / 1.4e15 * 1e6, 1)
        out[name] = r
    # bias + residual (the attention / MLP output projections), TF32 and bf16 operands
    for name, (M, N, Kd) in {"c2 o_proj": (4096, 768, 768), "c2 mlp_proj": (4096, 768, 3072),
                             "xl mlp_proj": (16384, 1600, 6400)}.items():
        A = torch.randn(M, Kd, device=dev)
        B = torch.randn(N, Kd, device=dev) * 0.05
        bias = torch.randn(N, device=dev)
        R = torch.randn(M, N, device=dev)
        C = torch.empty(M, N, device=dev)
        A16, B16 = A.to(torch.bfloat16), B.to(torch.bfloat16)
        out[name] = {"tf32_bias_res": timeit(lambda: K.gemm(A, B, C=C, bias=bias, R=R)),
                     "bf16_bias_res": timeit(lambda: K.gemm_bf16(A16, B16, C=C, bias=bias, R=R)),
                     "bf16_plain": timeit(lambda: K.gemm_bf16(A16, B16, C=C))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
