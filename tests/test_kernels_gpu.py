"""GPU parity of each sm_100a kernel against a plain PyTorch fp32 reference of the op.

Tolerances: the GEMM runs tcgen05 kind::tf32 (10-bit mantissa inputs, fp32 accumulate),
so GEMM-derived outputs are checked with relative Frobenius error <= 3e-3 against fp32;
everything else is fp32 CUDA-core math checked at <= 1e-4 relative (1e-5 absolute).
"""
import math

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2110_08633_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda:0")
torch.backends.cuda.matmul.allow_tf32 = False


def rel(a, b):
    return ((a - b).norm() / (b.norm() + 1e-30)).item()


SHAPES = [(128, 128, 32), (256, 384, 768), (300, 200, 96), (1024, 2304, 768), (4096, 768, 3072), (64, 1000, 64),
          (96, 520, 40)]


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_majors(shape, a_mn, b_mn):
    M, N, Kd = shape
    torch.manual_seed(M + N + Kd)
    A = torch.randn(M, Kd, device=dev)
    B = torch.randn(N, Kd, device=dev)
    ref = A @ B.T
    Ain = A.T.contiguous() if a_mn else A
    Bin = B.T.contiguous() if b_mn else B
    C = K.gemm(Ain, Bin, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=Kd)
    torch.cuda.synchronize()
    assert rel(C, ref) < 3e-3, (shape, a_mn, b_mn, rel(C, ref))


@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True), (True, False)])
def test_gemm_precision_fp32(a_mn, b_mn):
    """3xTF32 split: ~fp32 accuracy (rel <= 2e-5 vs an fp64 product; TF32 alone ~5e-4)."""
    M, N, Kd = 384, 256, 1024
    A = torch.randn(M, Kd, device=dev)
    B = torch.randn(N, Kd, device=dev)
    ref = (A.double() @ B.double().T)
    try:
        K.gemm_config(precision_fp32=True)
        C = K.gemm(A.T.contiguous() if a_mn else A, B.T.contiguous() if b_mn else B, a_mn=a_mn, b_mn=b_mn,
                   M=M, N=N, K=Kd)
    finally:
        K.gemm_config(precision_fp32=False)
    assert rel(C.double(), ref) < 2e-5
    C32 = K.gemm(A, B)
    assert rel(C32.double(), ref) > 1e-5  # plain TF32 is measurably coarser


@pytest.mark.parametrize("M,N,Kd,b_mn,a_mn", [(500, 768, 50257, True, False), (768, 768, 4096, True, True),
                                              (96, 200, 8192, False, False)])
def test_gemm_splitk(M, N, Kd, b_mn, a_mn):
    """Low-occupancy GEMMs split K through the workspace; deterministic fixed-order reduce."""
    Kp = (Kd + 127) // 128 * 128  # 16-byte row strides (the LM head pads V to 50304)
    Apad = torch.zeros(M, Kp, device=dev)
    Apad[:, :Kd] = torch.randn(M, Kd, device=dev) * 0.1
    A = Apad[:, :Kd]
    B = torch.randn(N, Kd, device=dev) * 0.1
    C0 = torch.randn(M, N, device=dev)
    ws = torch.empty(4 << 20, device=dev)
    try:
        K.gemm_config(splitk_ws=ws)
        Ain = A.T.contiguous() if a_mn else Apad
        Bin = B.T.contiguous() if b_mn else B
        lda = Ain.stride(0)
        C = K.gemm(Ain, Bin, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=Kd, C=C0.clone(), beta=1.0, lda=lda)
        C2 = K.gemm(Ain, Bin, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=Kd, C=C0.clone(), beta=1.0, lda=lda)
    finally:
        K.gemm_config()
    assert rel(C, C0 + A @ B.T) < 3e-3
    assert torch.equal(C, C2)


DW_SHAPES = [(3072, 768, 4096), (2304, 768, 4096), (768, 3072, 4096), (768, 2304, 4096), (768, 768, 4096),
             (6400, 1600, 1024), (1600, 6400, 1024)]


@pytest.mark.parametrize("a_mn", [False, True])
@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("shape", DW_SHAPES)
def test_gemm_split256_weight_grads(shape, a_mn, b_mn):
    """The weight-gradient shapes of C2 (K = 4096 tokens) and XL b2 (K = 1024) through the
    256-wide CTA-pair split-K path (taken when a workspace is set: the executor's default),
    beta = 1 accumulation into an existing gradient: equal to torch fp32 within the TF32 bound,
    equal to the unsplit kernel within TF32 rounding of the partial sums, and bitwise
    deterministic across calls."""
    M, N, Kd = shape
    torch.manual_seed(M * 7 + N + Kd)
    A = torch.randn(M, Kd, device=dev) * 0.1
    B = torch.randn(N, Kd, device=dev) * 0.1
    C0 = torch.randn(M, N, device=dev)
    Ain = A.T.contiguous() if a_mn else A
    Bin = B.T.contiguous() if b_mn else B
    ws = torch.empty(2 * 3072 * 768 + 16, device=dev)  # the executor's C2 split-K workspace size
    try:
        K.gemm_config(splitk_ws=ws)
        C1 = K.gemm(Ain, Bin, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=Kd, C=C0.clone(), beta=1.0)
        C2 = K.gemm(Ain, Bin, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=Kd, C=C0.clone(), beta=1.0)
    finally:
        K.gemm_config()
    Cu = K.gemm(Ain, Bin, a_mn=a_mn, b_mn=b_mn, M=M, N=N, K=Kd, C=C0.clone(), beta=1.0)  # no workspace: unsplit
    torch.cuda.synchronize()
    ref = C0 + A @ B.T
    assert rel(C1, ref) < 3e-3, rel(C1, ref)
    assert rel(C1 - C0, Cu - C0) < 1e-4  # same TF32 operands, fp32 partial sums in another order
    assert torch.equal(C1, C2)


def test_gemm_epilogues():
    M, N, Kd = 512, 640, 256
    A = torch.randn(M, Kd, device=dev)
    B = torch.randn(N, Kd, device=dev) * 0.05
    bias = torch.randn(N, device=dev)
    R = torch.randn(M, N, device=dev)
    C0 = torch.randn(M, N, device=dev)
    base = A @ B.T
    C = K.gemm(A, B, bias=bias, R=R)
    assert rel(C, base + bias + R) < 3e-3
    C2 = C0.clone()
    K.gemm(A, B, C=C2, beta=1.0)
    assert rel(C2, C0 + base) < 3e-3
    # GELU: C = gelu(pre), H = gelu'(pre) (stored for the backward)
    H = torch.empty(M, N, device=dev)
    G = K.gemm(A, B, bias=bias, mode=1, H=H)
    pre = (base + bias).clone().requires_grad_(True)
    gl = torch.nn.functional.gelu(pre, approximate="tanh")
    gl.backward(torch.ones_like(gl))
    assert rel(G, gl.detach()) < 3e-3
    assert rel(H, pre.grad) < 3e-3
    # GELU backward: C = acc * Hin
    Hin = torch.randn(M, N, device=dev)
    D = K.gemm(A, B, mode=2, H=Hin)
    assert rel(D, base * Hin) < 3e-3


def test_gemm_vocab_head_shapes():
    rows, d, V, Vp = 256, 128, 50257, 50304
    z = torch.randn(rows, d, device=dev)
    wte = torch.randn(V, d, device=dev) * 0.02
    logits = torch.zeros(rows, Vp, device=dev)
    K.gemm(z, wte, C=logits, M=rows, N=V, K=d, ldc=Vp)
    assert rel(logits[:, :V], z @ wte.T) < 3e-3
    assert logits[:, V:].abs().max().item() == 0
    # dz = dlogits @ wte (A K-major with K = V ragged; B MN-major)
    dl = torch.randn(rows, Vp, device=dev)
    dl[:, V:] = 0
    dz = K.gemm(dl, wte, a_mn=False, b_mn=True, M=rows, N=d, K=V, lda=Vp)
    assert rel(dz, dl[:, :V] @ wte) < 3e-3
    # dwte = dlogits^T @ z (both MN-major), M = V ragged
    dwte = torch.zeros(V, d, device=dev)
    K.gemm(dl, z, a_mn=True, b_mn=True, M=V, N=d, K=rows, lda=Vp, C=dwte)
    assert rel(dwte, dl[:, :V].T @ z) < 3e-3


@pytest.mark.parametrize("d", [64, 768, 1600, 4096])
def test_layernorm(d):
    rows = 333
    x = torch.randn(rows, d, device=dev) * 3 + 1
    g = torch.randn(d, device=dev)
    b = torch.randn(d, device=dev)
    y, mean, rstd = K.layernorm_fwd(x, g, b)
    ref = torch.nn.functional.layer_norm(x, (d,), g, b, 1e-5)
    assert rel(y, ref) < 1e-5
    xr = x.clone().requires_grad_(True)
    gr = g.clone().requires_grad_(True)
    br = b.clone().requires_grad_(True)
    dy = torch.randn(rows, d, device=dev)
    torch.nn.functional.layer_norm(xr, (d,), gr, br, 1e-5).backward(dy)
    prior = torch.randn(rows, d, device=dev)
    dx, dg, db = K.layernorm_bwd(x, g, mean, rstd, dy, dx=prior.clone(), accumulate=True)
    assert rel(dx, xr.grad + prior) < 1e-5
    assert rel(dg, gr.grad) < 1e-5
    assert rel(db, br.grad) < 1e-5


def ref_attention(qkv, B, T, H):
    D = H * 64
    q, k, v = qkv.view(B, T, 3, H, 64).permute(2, 0, 3, 1, 4)
    att = (q @ k.transpose(-1, -2)) / 8.0
    mask = torch.ones(T, T, device=qkv.device, dtype=torch.bool).tril()
    att = att.masked_fill(~mask, float("-inf")).softmax(-1)
    return (att @ v).permute(0, 2, 1, 3).reshape(B * T, D)


@pytest.mark.parametrize("B,T,H,chunk", [(2, 32, 1, None), (2, 100, 3, None), (1, 512, 2, None),
                                         (4, 128, 12, None), (8, 512, 12, 2), (2, 384, 4, 3), (3, 200, 5, 7)])
def test_attention(B, T, H, chunk):
    torch.manual_seed(T + H)
    qkv = torch.randn(B * T, 3 * H * 64, device=dev)
    wf = None if chunk is None else chunk * T * T  # forces (batch, head) chunking
    out = K.attention_fwd(qkv, B, T, H, work_floats=wf)
    qr = qkv.clone().requires_grad_(True)
    ref = ref_attention(qr, B, T, H)
    assert rel(out, ref) < 3e-3
    dout = torch.randn_like(out)
    ref.backward(dout)
    dqkv = K.attention_bwd(qkv, dout, B, T, H, work_floats=None if chunk is None else 2 * chunk * T * T)
    assert rel(dqkv, qr.grad) < 3e-3


@pytest.mark.parametrize("B,T,H", [(2, 32, 1), (2, 100, 3), (1, 512, 2), (4, 128, 12), (8, 512, 12), (2, 384, 4),
                                   (3, 200, 5), (1, 1024, 2)])
def test_flash_attention(B, T, H):
    """Fused tcgen05 attention (the TF32 path): forward, lse, and the dK/dV + dQ backward
    against PyTorch fp32 autograd; ragged T (not a multiple of the 128 / 64 tiles)."""
    torch.manual_seed(7 * T + H)
    qkv = torch.randn(B * T, 3 * H * 64, device=dev)
    out, lse = K.flash_attention_fwd(qkv, B, T, H)
    qr = qkv.clone().requires_grad_(True)
    ref = ref_attention(qr, B, T, H)
    assert rel(out, ref) < 3e-3
    q, k, _ = qkv.view(B, T, 3, H, 64).permute(2, 0, 3, 1, 4)
    s = (q @ k.transpose(-1, -2)) / 8.0
    s = s.masked_fill(~torch.ones(T, T, device=dev, dtype=torch.bool).tril(), float("-inf"))
    lse_ref = torch.logsumexp(s, -1).reshape(-1) / math.log(2.0)
    assert (lse - lse_ref).abs().max().item() < 2e-2
    dout = torch.randn_like(out)
    ref.backward(dout)
    dqkv = K.flash_attention_bwd(qkv, out, dout, lse, B, T, H)
    assert rel(dqkv, qr.grad) < 3e-3
    # deterministic (no atomics): bit-identical on a rerun
    assert torch.equal(dqkv, K.flash_attention_bwd(qkv, out, dout, lse, B, T, H))


def test_embedding():
    V, d, B, T = 1000, 128, 3, 40
    tok = torch.randint(0, V, (B * T,), device=dev, dtype=torch.int32)
    tok[:10] = 5  # collisions
    wte = torch.randn(V, d, device=dev)
    wpe = torch.randn(T, d, device=dev)
    h = K.embed_fwd(tok, wte, wpe, T)
    pos = torch.arange(B * T, device=dev) % T
    assert rel(h, wte[tok.long()] + wpe[pos]) < 1e-6
    dh = torch.randn(B * T, d, device=dev)
    dwte, dwpe = K.embed_bwd(tok, dh, V, T)
    ref_wte = torch.zeros(V, d, device=dev).index_add_(0, tok.long(), dh)
    assert rel(dwte, ref_wte) < 1e-5
    assert rel(dwpe, dh.view(B, T, d).sum(0)) < 1e-5


@pytest.mark.parametrize("V,Vp", [(50257, 50304), (1000, 1003), (30001, 30004)])
def test_softmax_xent(V, Vp):
    """Register-resident path (16-byte aligned rows, V & 3 tail), and the 3-pass fallback
    (unaligned row stride)."""
    rows = 77
    logits = torch.randn(rows, Vp, device=dev) * 3
    tgt = torch.randint(0, V, (rows,), device=dev, dtype=torch.int32)
    lr = logits[:, :V].clone().requires_grad_(True)
    loss = torch.nn.functional.cross_entropy(lr, tgt.long(), reduction="none")
    loss.sum().backward()
    scale = 1.0 / 300
    row_loss = K.softmax_xent(logits, tgt, V, scale)
    assert rel(row_loss, loss.detach()) < 1e-5
    assert rel(logits[:, :V], lr.grad * scale) < 1e-4


def test_bias_grad_and_adam():
    dy = torch.randn(3000, 700, device=dev)
    assert rel(K.bias_grad(dy), dy.sum(0)) < 1e-5
    n = 1 << 16
    p = torch.randn(n, device=dev)
    g = torch.randn(n, device=dev)
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    pr = p.clone().requires_grad_(True)
    opt = torch.optim.Adam([pr], lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    for step in range(1, 4):
        K.adam(p, g, m, v, 1e-3, step)
        pr.grad = g.clone()
        opt.step()
    assert rel(p, pr.detach()) < 1e-6


@pytest.mark.parametrize("bf16", [False, True])
def test_adam_host_state_zero_copy(bf16):
    """The executor's GPU-side optimizer: moments in pinned host memory read/written by the
    kernel over the link; must equal the HBM-resident Adam (same arithmetic)."""
    n = (1 << 20) + 96
    p = torch.randn(n, device=dev) * 0.02
    p_ref = p.clone()
    mdt = torch.bfloat16 if bf16 else torch.float32
    m_h = torch.zeros(n, dtype=mdt).pin_memory()
    v_h = torch.zeros(n, dtype=mdt).pin_memory()
    p_h = torch.empty(n).pin_memory()
    m_r = torch.zeros(n, device=dev)
    v_r = torch.zeros(n, device=dev)
    for step in range(1, 4):
        g = torch.randn(n, device=dev) * 1e-3
        K.adam_host_state(p, g, m_h, v_h, p_h, 1e-3, step, weight_decay=0.01)
        K.adam(p_ref, g, m_r, v_r, 1e-3, step, weight_decay=0.01)
        if bf16:  # the reference emulation: moments rounded to bf16 after each update
            m_r.copy_(m_r.bfloat16().float())
            v_r.copy_(v_r.bfloat16().float())
    torch.cuda.synchronize()
    assert torch.equal(p_h.to(dev), p)
    if bf16:
        assert rel(p, p_ref) < 1e-5
        assert rel(m_h.to(dev).float(), m_r) < 1e-2
    else:
        assert torch.equal(p, p_ref)
        assert torch.equal(m_h.to(dev), m_r) and torch.equal(v_h.to(dev), v_r)
