"""Pinning the CPU numeric oracle (oracle/gpt_oracle.c).

The reference never executes tensors, so the oracle is pinned against an
independent restatement: PyTorch CPU autograd in float64 of the same GPT-2 (same flat
parameter vector, include/hydra_gpt.h). Also: sharded execution == unsharded execution
(the reference's claim that checkpoint+recompute does not change training).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402


def torch_gpt_loss(m, params, tok, tgt):
    """Float64 autograd restatement of the model in include/hydra_gpt.h."""
    P = torch.tensor(params, dtype=torch.float64, requires_grad=True)
    d, V, T, B, H = m.d, m.V, m.T, m.B, m.H

    def seg(off, n, shape):
        return P[off:off + n].view(*shape)

    wte = seg(0, V * d, (V, d))
    wpe = seg(O.pad32(V * d), T * d, (T, d))
    x = wte[torch.tensor(tok, dtype=torch.long)] + wpe.repeat(B, 1)
    sizes = [d, d, 3 * d * d, 3 * d, d * d, d, d, d, 4 * d * d, 4 * d, 4 * d * d, d]
    shapes = [(d,), (d,), (3 * d, d), (3 * d,), (d, d), (d,), (d,), (d,), (4 * d, d), (4 * d,), (d, 4 * d), (d,)]
    mask = torch.ones(T, T, dtype=torch.bool).tril()
    for l in range(1, m.L + 1):
        off = O.layer_offset(m, l)
        t = []
        for s, sh in zip(sizes, shapes):
            t.append(seg(off, s, sh))
            off += O.pad32(s)
        g1, b1, wqkv, bqkv, wo, bo, g2, b2, wfc, bfc, wpr, bpr = t
        a = torch.nn.functional.layer_norm(x, (d,), g1, b1, 1e-5)
        qkv = a @ wqkv.T + bqkv
        q, k, v = qkv.view(B, T, 3, H, 64).permute(2, 0, 3, 1, 4)
        att = ((q @ k.transpose(-1, -2)) / 8.0).masked_fill(~mask, float("-inf")).softmax(-1)
        y = (att @ v).permute(0, 2, 1, 3).reshape(B * T, d)
        x = x + y @ wo.T + bo
        a = torch.nn.functional.layer_norm(x, (d,), g2, b2, 1e-5)
        hmid = torch.nn.functional.gelu(a @ wfc.T + bfc, approximate="tanh")
        x = x + hmid @ wpr.T + bpr
    off = O.layer_offset(m, m.L + 1)
    z = torch.nn.functional.layer_norm(x, (d,), seg(off, d, (d,)), seg(off + O.pad32(d), d, (d,)), 1e-5)
    loss = torch.nn.functional.cross_entropy(z @ wte.T, torch.tensor(tgt, dtype=torch.long))
    loss.backward()
    return loss.item(), P.grad.numpy()


@pytest.fixture(scope="module")
def tiny():
    m = O.make_dims(d=64, L=2, T=16, B=2)
    params = O.init_params(m, 1234)
    tok, tgt = O.tokens(m, 7, 0, 0)
    return m, params, tok, tgt


def test_tokens_in_range_and_deterministic(tiny):
    m, _, tok, tgt = tiny
    assert tok.min() >= 0 and tok.max() < 50257
    assert np.array_equal(tok[1:m.T], tgt[:m.T - 1])  # targets are the shifted stream
    tok2, _ = O.tokens(m, 7, 0, 0)
    assert np.array_equal(tok, tok2)
    tok3, _ = O.tokens(m, 7, 0, 1)
    assert not np.array_equal(tok, tok3)


def test_init_statistics(tiny):
    m, params, _, _ = tiny
    wte = params[: m.V * m.d]
    assert abs(wte.std() - 0.02) < 1e-3 and abs(wte.mean()) < 1e-3
    off = O.layer_offset(m, m.L + 1)
    assert np.all(params[off: off + m.d] == 1.0)


def test_oracle_matches_torch_float64(tiny):
    m, params, tok, tgt = tiny
    loss_ref, grad_ref = torch_gpt_loss(m, params, tok, tgt)
    grads = np.zeros_like(params)
    _, loss = O.shard_fwd(m, params, 0, m.L + 2, tok, tgt, None)
    O.shard_bwd(m, params, grads, 0, m.L + 2, tok, tgt, None, None)
    assert abs(loss - loss_ref) / loss_ref < 1e-6
    for l in range(m.L + 2):
        a, b = O.layer_offset(m, l), O.layer_offset(m, l + 1)
        rel = np.linalg.norm(grads[a:b] - grad_ref[a:b]) / (np.linalg.norm(grad_ref[a:b]) + 1e-30)
        assert rel < 1e-5, (l, rel)


@pytest.mark.parametrize("starts", [[0, 2], [0, 1, 3], [0, 3], [0, 1, 2, 3]])
def test_sharded_equals_unsharded(tiny, starts):
    m, params0, tok, tgt = tiny
    p_a, p_b = params0.copy(), params0.copy()
    ma, va = np.zeros_like(p_a), np.zeros_like(p_a)
    mb_, vb = np.zeros_like(p_b), np.zeros_like(p_b)
    for step in (1, 2):
        la = O.sharded_step(m, p_a, ma, va, [0], step, 1e-3, tok, tgt)
        lb = O.sharded_step(m, p_b, mb_, vb, starts, step, 1e-3, tok, tgt)
        assert la == lb
    assert np.array_equal(p_a, p_b)


def test_bf16_state_rounding_is_rne():
    p = np.zeros(4, dtype=np.float32)
    g = np.array([1.0, -3.0, 1e-3, 7.7], dtype=np.float32)
    m = np.zeros(4, dtype=np.float32)
    v = np.zeros(4, dtype=np.float32)
    O.adam(p, g, m, v, 1e-3, 1, bf16_state=True)
    for x in np.concatenate([m, v]):
        bits = np.array([x], dtype=np.float32).view(np.uint32)[0]
        assert bits & 0xFFFF == 0  # representable in bfloat16
    assert abs(m[3] - 0.77) / 0.77 < 1 / 128
