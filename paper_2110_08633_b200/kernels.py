"""Tensor-level wrappers over the C-ABI kernel entry points (include/hydra.h).

Used by the GPU parity tests and by tools; tensors are fp32 CUDA tensors (row-major,
contiguous unless a leading dimension is given). Every call goes to libhydra.so — the
sm_100a kernels — on torch's current stream.
"""
import torch

from ._lib import check, lib


def _s():
    return ctypes_stream(torch.cuda.current_stream())


def ctypes_stream(stream):
    return stream.cuda_stream


def _p(t):
    return None if t is None else t.data_ptr()


def gemm_config(precision_fp32=False, splitk_ws=None):
    """Per-thread GEMM settings: 3xTF32 ("fp32") precision and the split-K workspace."""
    check(lib().hy_gemm_config(int(precision_fp32), _p(splitk_ws), 0 if splitk_ws is None else splitk_ws.numel()))


def gemm(A, B, *, a_mn=False, b_mn=False, M=None, N=None, K=None, C=None, bias=None, R=None, beta=0.0,
         mode=0, H=None, lda=None, ldb=None, ldc=None):
    """C = op(A) op(B)^T. a_mn=False: A is [M,K]; True: A is [K,M]. Likewise B with N."""
    if not a_mn:
        M_, K_ = A.shape
    else:
        K_, M_ = A.shape
    if not b_mn:
        N_ = B.shape[0]
    else:
        N_ = B.shape[1]
    M = M or M_
    K = K or K_
    N = N or N_
    if C is None:
        C = torch.empty(M, N, device=A.device, dtype=torch.float32)
    lda = lda or A.stride(0)
    ldb = ldb or B.stride(0)
    ldc = ldc or C.stride(0)
    ldr = R.stride(0) if R is not None else 0
    ldh = H.stride(0) if H is not None else 0
    hout = H if mode == 1 else None
    hin = H if mode == 2 else None
    check(lib().hy_gemm(_s(), M, N, K, _p(A), lda, int(a_mn), _p(B), ldb, int(b_mn), _p(C), ldc, _p(bias), _p(R), ldr,
                        float(beta), int(mode), _p(hout), _p(hin), ldh))
    return C


def gemm_bf16(A, B, *, a_mn=False, b_mn=False, C=None, c_bf16=False, bias=None, R=None, beta=0.0, mode=0, H=None):
    """bf16-operand GEMM (tcgen05 kind::f16, fp32 accumulate): C = op(A) op(B)^T (+ epilogue).
    A, B: torch.bfloat16 CUDA tensors; C fp32, or bf16 when c_bf16."""
    assert A.dtype == torch.bfloat16 and B.dtype == torch.bfloat16
    M, K = (A.shape[1], A.shape[0]) if a_mn else (A.shape[0], A.shape[1])
    N = B.shape[1] if b_mn else B.shape[0]
    if C is None:
        C = torch.empty(M, N, device=A.device, dtype=torch.bfloat16 if c_bf16 else torch.float32)
    ldr = R.stride(0) if R is not None else 0
    ldh = H.stride(0) if H is not None else 0
    hout = H if mode == 1 else None
    hin = H if mode == 2 else None
    check(lib().hy_gemm_bf16(_s(), M, N, K, _p(A), A.stride(0), int(a_mn), _p(B), B.stride(0), int(b_mn), _p(C),
                             C.stride(0), int(c_bf16), _p(bias), _p(R), ldr, float(beta), int(mode), _p(hout),
                             _p(hin), ldh))
    return C


def to_bf16(x):
    y = torch.empty(x.shape, device=x.device, dtype=torch.bfloat16)
    check(lib().hy_to_bf16(_s(), x.numel(), _p(x), _p(y)))
    return y


def layernorm_fwd(x, g, b):
    rows, d = x.shape
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=x.device)
    rstd = torch.empty(rows, device=x.device)
    check(lib().hy_layernorm_fwd(_s(), rows, d, _p(x), _p(g), _p(b), _p(y), _p(mean), _p(rstd)))
    return y, mean, rstd


def layernorm_bwd(x, g, mean, rstd, dy, dx=None, accumulate=False):
    rows, d = x.shape
    if dx is None:
        dx = torch.zeros_like(x)
    dg = torch.zeros(d, device=x.device)
    db = torch.zeros(d, device=x.device)
    ws = torch.empty(2 * d * 400, device=x.device)
    check(lib().hy_layernorm_bwd(_s(), rows, d, _p(x), _p(g), _p(mean), _p(rstd), _p(dy), _p(dx), int(accumulate),
                                 _p(dg), _p(db), _p(ws)))
    return dx, dg, db


def attention_fwd(qkv, B, T, H, work_floats=None):
    out = torch.empty(B * T, H * 64, device=qkv.device)
    wf = work_floats or B * H * T * T
    work = torch.empty(wf, device=qkv.device)
    check(lib().hy_attention_fwd(_s(), B, T, H, 64, _p(qkv), _p(out), _p(work), wf))
    return out


def attention_bwd(qkv, dout, B, T, H, work_floats=None):
    dqkv = torch.empty_like(qkv)
    wf = work_floats or 2 * B * H * T * T
    work = torch.empty(wf, device=qkv.device)
    check(lib().hy_attention_bwd(_s(), B, T, H, 64, _p(qkv), _p(dout), _p(dqkv), _p(work), wf))
    return dqkv


def flash_attention_fwd(qkv, B, T, H):
    out = torch.empty(B * T, H * 64, device=qkv.device)
    lse = torch.empty(B * H * T, device=qkv.device)
    check(lib().hy_flash_attention_fwd(_s(), B, T, H, _p(qkv), _p(out), _p(lse)))
    return out, lse


def flash_attention_bwd(qkv, out, dout, lse, B, T, H):
    dqkv = torch.empty_like(qkv)
    di = torch.empty(B * H * T, device=qkv.device)
    check(lib().hy_flash_attention_bwd(_s(), B, T, H, _p(qkv), _p(out), _p(dout), _p(lse), _p(dqkv), _p(di)))
    return dqkv


def embed_fwd(tokens, wte, wpe, T):
    rows = tokens.numel()
    d = wte.shape[1]
    h = torch.empty(rows, d, device=wte.device)
    check(lib().hy_embed_fwd(_s(), rows, T, d, _p(tokens), _p(wte), _p(wpe), _p(h)))
    return h


def embed_bwd(tokens, dh, V, T, dwte=None):
    rows, d = dh.shape
    if dwte is None:
        dwte = torch.zeros(V, d, device=dh.device)
    dwpe = torch.empty(T, d, device=dh.device)
    check(lib().hy_embed_bwd(_s(), rows, T, d, V, _p(tokens), _p(dh), _p(dwte), _p(dwpe)))
    return dwte, dwpe


def softmax_xent(logits, targets, V, grad_scale):
    rows = logits.shape[0]
    row_loss = torch.empty(rows, device=logits.device)
    check(lib().hy_softmax_xent(_s(), rows, V, _p(logits), logits.stride(0), _p(targets), float(grad_scale),
                                _p(row_loss)))
    return row_loss


def bias_grad(dy, out=None, accumulate=False):
    M, N = dy.shape
    if out is None:
        out = torch.zeros(N, device=dy.device)
    ws = torch.empty(N * 400, device=dy.device)
    check(lib().hy_bias_grad(_s(), M, N, _p(dy), dy.stride(0), _p(out), int(accumulate), _p(ws)))
    return out


def adam(p, g, m, v, lr, step, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
    check(lib().hy_adam(_s(), p.numel(), _p(p), _p(g), _p(m), _p(v), lr, beta1, beta2, eps, weight_decay, step))


def adam_host_state(p, g, m_host, v_host, p_host, lr, step, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0,
                    grid=0):
    """Zero-copy AdamW: p, g on the GPU; m, v, p_host pinned host tensors (fp32, or bf16 moments)."""
    bf16 = int(m_host.dtype == torch.bfloat16)
    check(lib().hy_adam_host_state(_s(), p.numel(), _p(p), _p(g), _p(m_host), _p(v_host), _p(p_host), lr, beta1,
                                   beta2, eps, weight_decay, step, bf16, grid))
