"""Time the tcgen05 GEMM at the workload's shapes for each tile width (CUDA events)."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {  # name: (M, N, K, a_mn, b_mn)
    "qkv fwd": (4096, 2304, 768, 0, 0), "o fwd": (4096, 768, 768, 0, 0), "fc fwd": (4096, 3072, 768, 0, 0),
    "pr fwd": (4096, 768, 3072, 0, 0), "dX(pr)": (4096, 3072, 768, 0, 1), "dW(pr)": (768, 3072, 4096, 1, 1),
    "dW(fc)": (3072, 768, 4096, 1, 1), "logits": (500, 50257, 768, 0, 0), "xl fc": (8192, 6400, 1600, 0, 0),
    "sq 8192": (8192, 8192, 8192, 0, 0),
}


def run(bn):
    import torch
    from paper_2110_08633_b200 import kernels as K
    dev = torch.device("cuda")
    out = {}
    for name, (M, N, Kd, amn, bmn) in SHAPES.items():
        A = torch.randn(Kd, M, device=dev) if amn else torch.randn(M, Kd, device=dev)
        ldb = None
        if name == "logits":
            B = torch.randn(N, Kd, device=dev)
            C = torch.empty(M, 50304, device=dev)
        else:
            B = torch.randn(Kd, N, device=dev) if bmn else torch.randn(N, Kd, device=dev)
            C = torch.empty(M, N, device=dev)
        f = lambda: K.gemm(A, B, a_mn=bool(amn), b_mn=bool(bmn), M=M, N=N, K=Kd, C=C, ldc=C.stride(0))
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        reps = 20
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps / 1e3
        out[name] = round(2.0 * M * N * Kd / t / 1e12, 1)
    return out


def run_cublas():
    """cuBLAS TF32 at the same shapes (torch.matmul, allow_tf32): the library yardstick."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = True
    dev = torch.device("cuda")
    out = {}
    for name, (M, N, Kd, amn, bmn) in SHAPES.items():
        A = torch.randn(Kd, M, device=dev).t() if amn else torch.randn(M, Kd, device=dev)
        B = torch.randn(Kd, N, device=dev) if bmn else torch.randn(N, Kd, device=dev).t()
        C = torch.empty(M, N, device=dev)
        f = lambda: torch.matmul(A, B, out=C)
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20 / 1e3
        out[name] = round(2.0 * M * N * Kd / t / 1e12, 1)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "cublas":
        print(json.dumps(run_cublas()))
    elif len(sys.argv) > 1:
        print(json.dumps(run(int(sys.argv[1]))))
    else:
        res = {}
        for bn in ("0", "nopair", "cublas"):
            env = dict(os.environ, HY_GEMM_BN=bn, HY_GEMM_PAIR="0" if bn == "nopair" else "1")
            bn = "0" if bn == "nopair" else bn
            r = subprocess.run([sys.executable, __file__, bn], env=env, capture_output=True, text=True, timeout=180)
            key = env["HY_GEMM_BN"]
            res[key] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
        print(json.dumps(res, indent=1))
