"""GPU parity of the bf16 precision's kernels (tcgen05 kind::f16 GEMM family, bf16 epilogue
stores, fp32 -> bf16 conversion, bf16 LayerNorm output / column sums) and of the executor's
bf16 path on toy dims against the bf16-emulating CPU oracle.

Reference for the GEMMs: torch fp32 matmul (TF32 off) of the same bf16 operands widened to fp32
— a bf16 x bf16 product is exact in fp32, so the two differ only in fp32 summation order
(relative Frobenius error <= 1e-5 here, against ~3e-3 for the TF32 kernels vs unrounded fp32).
"""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2110_08633_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False


def rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-30)).item()


def bf(x):
    return x.to(torch.bfloat16)


# (M, N, K): one-CTA tiles (M <= 128), CTA pairs with BN 128 / 192 / 256, ragged edges, the
# GPT-2 small / XL block shapes; every stride a multiple of 8 bf16 (16-byte TMA rows).
SHAPES = [(128, 128, 64), (256, 384, 768), (304, 200, 96), (1024, 2304, 768), (4096, 768, 3072), (64, 1000, 64),
          (96, 520, 40), (2048, 6400, 1600), (520, 3072, 768)]


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_bf16_majors(shape, a_mn, b_mn):
    M, N, Kd = shape
    torch.manual_seed(M + 3 * N + Kd)
    A = bf(torch.randn(M, Kd, device=dev))
    B = bf(torch.randn(N, Kd, device=dev))
    ref = A.float() @ B.float().T
    C = K.gemm_bf16(A.T.contiguous() if a_mn else A, B.T.contiguous() if b_mn else B, a_mn=a_mn, b_mn=b_mn)
    torch.cuda.synchronize()
    assert C.shape == (M, N)
    assert rel(C, ref) < 1e-5, (shape, a_mn, b_mn, rel(C, ref))


@pytest.mark.parametrize("a_mn,b_mn", [(True, True), (False, True), (True, False)])
@pytest.mark.parametrize("shape", [(3072, 768, 4096), (2304, 768, 4096), (768, 3072, 4096), (768, 768, 4096),
                                   (6400, 1600, 1024), (1600, 6400, 1024), (768, 768, 50304)])
def test_gemm_bf16_splitk_weight_grads(shape, a_mn, b_mn):
    """The weight-gradient shapes (K = tokens) take split-K through the workspace (256-wide pair
    tiles or the low-occupancy split), beta = 1 into an existing gradient: equal to torch within
    fp32 summation order, to the unsplit kernel within partial-sum reordering, and bitwise
    deterministic across calls."""
    M, N, Kd = shape
    torch.manual_seed(M + N + 5 * Kd)
    A = bf(torch.randn(M, Kd, device=dev) * 0.1)
    B = bf(torch.randn(N, Kd, device=dev) * 0.1)
    C0 = torch.randn(M, N, device=dev)
    Ain = A.T.contiguous() if a_mn else A
    Bin = B.T.contiguous() if b_mn else B
    ws = torch.empty(2 * 3072 * 768 + 16, device=dev)
    try:
        K.gemm_config(splitk_ws=ws)
        C1 = K.gemm_bf16(Ain, Bin, a_mn=a_mn, b_mn=b_mn, C=C0.clone(), beta=1.0)
        C2 = K.gemm_bf16(Ain, Bin, a_mn=a_mn, b_mn=b_mn, C=C0.clone(), beta=1.0)
    finally:
        K.gemm_config()
    Cu = K.gemm_bf16(Ain, Bin, a_mn=a_mn, b_mn=b_mn, C=C0.clone(), beta=1.0)
    torch.cuda.synchronize()
    ref = (C0.double() + A.double() @ B.double().T).float()  # fp64: K up to 50304 terms
    assert rel(C1, ref) < 2e-5, rel(C1, ref)
    # the unsplit kernel sums all K in one fp32 TMEM accumulator: ~sqrt(K) 2^-24 drift at K = 50304
    assert rel(C1 - C0, Cu - C0) < (1e-4 if Kd > 8192 else 1e-5)
    assert torch.equal(C1, C2)


@pytest.mark.parametrize("M", [512, 4096])
def test_gemm_bf16_epilogues(M):
    N, Kd = 640, 256
    torch.manual_seed(M)
    A = bf(torch.randn(M, Kd, device=dev))
    B = bf(torch.randn(N, Kd, device=dev) * 0.05)
    bias = torch.randn(N, device=dev)
    R = torch.randn(M, N, device=dev)
    base = A.float() @ B.float().T
    # store + bias + residual (fp32 C)
    C = K.gemm_bf16(A, B, bias=bias, R=R)
    assert rel(C, base + bias + R) < 1e-5
    # GELU forward: bf16 activation out, fp32 gelu'(pre-activation) for the backward
    H = torch.empty(M, N, device=dev)
    G = K.gemm_bf16(A, B, bias=bias, mode=1, H=H, c_bf16=True)
    assert G.dtype == torch.bfloat16
    h = base + bias
    hd = h.clone().requires_grad_(True)
    torch.nn.functional.gelu(hd, approximate="tanh").backward(torch.ones_like(h))
    assert rel(H, hd.grad) < 1e-5
    g_ref = torch.nn.functional.gelu(h, approximate="tanh")
    # bf16 rounding of the output: <= 2^-9 relative per element
    assert rel(G, g_ref) < 4e-3
    assert ((G.float() - g_ref).abs() <= g_ref.abs() * 2.0 ** -8 + 1e-6).float().mean().item() > 0.999
    # GELU backward: C = acc * H (the stored gelu') as bf16
    D = K.gemm_bf16(A, B, mode=2, H=H, c_bf16=True)
    assert rel(D, base * hd.grad) < 4e-3


def test_to_bf16_is_rne():
    x = torch.randn(1 << 20, device=dev) * 3
    x[:8] = torch.tensor([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, -0.0, 65504.0, 1e-40, float("inf"), -1e30, 0.5],
                         device=dev)
    y = K.to_bf16(x)
    assert torch.equal(y.view(torch.int16), x.to(torch.bfloat16).view(torch.int16))


def test_executor_bf16_toy_vs_oracle(tmp_path):
    """Two-shard toy job in the bf16 precision against the oracle in its bf16 mode (same
    operands rounded): losses and parameters within the bf16 bound of tests/
    test_baseline_shapes_gpu.py, and measurably off the fp32 oracle (the rounding is real)."""
    import numpy as np

    import paper_2110_08633_b200 as P
    from oracle import oracle as O
    from test_executor_gpu import tiny_config

    cfg = tiny_config(mem=50e6)
    starts = [[0, 3]] * len(cfg["jobs"])
    ex = P.Executor(cfg, gpus=1, passes=1, precision="bf16")
    try:
        res = ex.run(1)
        gp = {j: ex.read_params(j) for j in range(len(cfg["jobs"]))}
    finally:
        ex.close()
    starts = res["shard_starts"]
    O.set_bf16(True)
    try:
        losses, params = O.run_workload_cpu(cfg, starts)
    finally:
        O.set_bf16(False)
    losses32, params32 = O.run_workload_cpu(cfg, starts)
    for j in losses:
        gl = np.array(res["losses"][j][: len(losses[j])])
        assert np.max(np.abs(gl - losses[j]) / np.abs(losses[j])) < 2e-3
        d16 = np.linalg.norm(gp[j] - params[j]) / np.linalg.norm(params[j])
        d32 = np.linalg.norm(params32[j] - params[j]) / np.linalg.norm(params[j])
        assert d16 < 4e-3, d16
        assert d16 < d32, (d16, d32)


@pytest.mark.parametrize("M,N,Kd", [(333, 200, 96), (4100, 3080, 768), (1000, 520, 256)])
def test_gemm_ragged_epilogues_both_precisions(M, N, Kd):
    """Ragged M / N through the CTA-pair kernel's epilogues (the TMA-store path clips the tile
    edges; bias columns past N are never read): store + bias, GELU (+ gelu') with fp32 and bf16
    outputs, GELU', for TF32 and bf16 operands."""
    torch.manual_seed(M + N)
    A = torch.randn(M, Kd, device=dev)
    B = torch.randn(N, Kd, device=dev) * 0.05
    bias = torch.randn(N, device=dev)
    for prec in ("tf32", "bf16"):
        if prec == "bf16":
            A_, B_ = bf(A), bf(B)
            base = A_.float() @ B_.float().T
            run = lambda **kw: K.gemm_bf16(A_, B_, **kw)  # noqa: E731
            tol = 1e-5
        else:
            base = A @ B.T
            run = lambda **kw: K.gemm(A, B, **kw)  # noqa: E731
            tol = 3e-3
        C = run(bias=bias)
        assert rel(C, base + bias) < tol, (prec, "bias")
        pre = (base + bias).clone().requires_grad_(True)
        gl = torch.nn.functional.gelu(pre, approximate="tanh")
        gl.backward(torch.ones_like(gl))
        G = run(bias=bias, mode=1)
        assert rel(G, gl.detach()) < max(tol, 1e-5) * 3, (prec, "gelu")
        H = torch.empty(M, N, device=dev)
        G2 = run(bias=bias, mode=1, H=H)
        assert rel(G2, gl.detach()) < max(tol, 1e-5) * 3 and rel(H, pre.grad) < max(tol, 1e-5) * 3, (prec, "gelu+h")
        if prec == "bf16":
            G16 = run(bias=bias, mode=1, c_bf16=True)
            assert rel(G16, gl.detach()) < 4e-3
        D = run(mode=2, H=H)
        assert rel(D, base * H) < max(tol, 1e-5) * 3, (prec, "gelu'")
