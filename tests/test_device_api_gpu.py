"""Device-level C-ABI (include/hydra.h "Device level", SURVEY §8b minimum exports): capped HBM
arena, lanes, pinned copies, events, and one shard task's forward / backward against the CPU
oracle (oracle/gpt_oracle.c shard_fwd / shard_bwd)."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2110_08633_b200 as P  # noqa: E402
from paper_2110_08633_b200 import _lib  # noqa: E402
from paper_2110_08633_b200 import kernels as K  # noqa: E402
from oracle import oracle as O  # noqa: E402

L = P.lib()
vp = ctypes.c_void_p


def ok(rc):
    if rc != 0:
        raise P.HydraError(rc, L.hy_last_error().decode())


class Dev:
    def __init__(self, budget):
        self.h = vp()
        ok(L.hy_open(0, budget, ctypes.byref(self.h)))

    def alloc(self, nbytes):
        p = vp()
        ok(L.hy_arena_alloc(self.h, nbytes, ctypes.byref(p)))
        return p.value

    def put(self, arr):
        a = np.ascontiguousarray(arr)
        p = self.alloc(a.nbytes)
        ok(L.hy_copy_h2d(self.h, p, a.ctypes.data, a.nbytes))
        ok(L.hy_lane_sync(self.h, 0))
        return p

    def get(self, p, like):
        out = np.empty_like(like)
        ok(L.hy_copy_d2h(self.h, out.ctypes.data, p, out.nbytes))
        ok(L.hy_lane_sync(self.h, 1))
        return out

    def close(self):
        L.hy_close(self.h)


def test_arena_budget_copies_events():
    d = Dev(64 << 20)
    a = d.alloc(48 << 20)
    with pytest.raises(P.HydraError) as e:
        d.alloc(32 << 20)  # beyond the cap
    assert e.value.code == -3  # HY_E_CAPACITY
    peak = ctypes.c_size_t()
    ok(L.hy_arena_peak(d.h, ctypes.byref(peak)))
    assert peak.value == 48 << 20
    host = vp()
    ok(L.hy_pinned_alloc(1 << 20, ctypes.byref(host)))
    src = np.frombuffer((ctypes.c_float * (1 << 18)).from_address(host.value), dtype=np.float32)
    src[:] = np.arange(1 << 18, dtype=np.float32)
    e0, e1 = vp(), vp()
    ok(L.hy_event_record(d.h, 0, ctypes.byref(e0)))
    ok(L.hy_copy_h2d(d.h, a, host.value, 1 << 20))
    ok(L.hy_event_record(d.h, 0, ctypes.byref(e1)))
    ok(L.hy_lane_wait(d.h, 1, e1))  # UP waits for DOWN's copy
    back = np.zeros(1 << 18, dtype=np.float32)
    ok(L.hy_copy_d2h(d.h, back.ctypes.data, a, 1 << 20))
    ok(L.hy_lane_sync(d.h, 1))
    assert np.array_equal(back, src)
    done, ms = ctypes.c_int(), ctypes.c_float()
    ok(L.hy_event_query(e1, ctypes.byref(done)))
    assert done.value == 1
    ok(L.hy_event_elapsed(e0, e1, ctypes.byref(ms)))
    assert ms.value >= 0
    for ev in (e0, e1):
        ok(L.hy_event_destroy(ev))
    ok(L.hy_pinned_free(host))
    d.close()


@pytest.mark.parametrize("split", [None, 2])
def test_shard_forward_backward_match_oracle(split):
    """GPT with 3 blocks (d 64) run as one shard [0, L+2) — forward loss and backward gradients
    vs the oracle — or as two shards (embed + 2 blocks | last block + head, tied wte passed
    separately) chained through act_out -> act_in, forward loss vs the oracle. 3xTF32."""
    m = O.make_dims(d=64, L=3, T=32, B=2)
    dims = _lib.Dims(m.V, m.d, m.L, m.T, m.B, m.H)
    params = O.init_params(m, O.model_key(7, 0))
    tok, tgt = O.tokens(m, 7, 0, 0)
    zeros = np.zeros(m.B * m.T * m.d, dtype=np.float32)
    _, loss_ref = O.shard_fwd(m, params, 0, m.L + 2, tok, tgt, zeros)
    K.gemm_config(precision_fp32=True)
    d = Dev(256 << 20)
    try:
        need = ctypes.c_size_t()
        ok(L.hy_shard_scratch_bytes(ctypes.byref(dims), m.L, ctypes.byref(need)))
        scratch = d.alloc(need.value)
        t_dev, g_dev = d.put(tok), d.put(tgt)
        loss = ctypes.c_double()
        if split is None:
            p_dev = d.put(params)
            grads = d.put(np.zeros_like(params))
            bufs = _lib.ShardBufs(params=p_dev, tokens=t_dev, targets=g_dev, grads=grads, scratch=scratch,
                                  scratch_bytes=need.value)
            desc = _lib.ShardDesc(dims, 0, m.L + 2)
            ok(L.hy_shard_forward(d.h, ctypes.byref(desc), ctypes.byref(bufs), ctypes.byref(loss)))
            assert abs(loss.value - loss_ref) / loss_ref < 1e-5
            ok(L.hy_shard_backward(d.h, ctypes.byref(desc), ctypes.byref(bufs), ctypes.byref(loss)))
            ok(L.hy_lane_sync(d.h, 2))
            g = d.get(grads, params)
            g_ref = np.zeros_like(params)
            O.shard_bwd(m, params, g_ref, 0, m.L + 2, tok, tgt, zeros, zeros)
            for layer in range(m.L + 2):
                lo, hi = O.layer_offset(m, layer), O.layer_offset(m, layer + 1)
                rel = np.linalg.norm(g[lo:hi] - g_ref[lo:hi]) / np.linalg.norm(g_ref[lo:hi])
                assert rel < 5e-4, (layer, rel)  # raw gradients: 3xTF32 vs fp64 accumulation
        else:
            cut = O.layer_offset(m, split + 1)  # layers [0, split+1) | [split+1, L+2)
            p0, p1 = d.put(params[:cut]), d.put(params[cut:])
            wte = d.put(params[:O.layer_offset(m, 1)])
            act = d.alloc(zeros.nbytes)
            b0 = _lib.ShardBufs(params=p0, tokens=t_dev, targets=g_dev, act_out=act, scratch=scratch,
                                scratch_bytes=need.value)
            ok(L.hy_shard_forward(d.h, ctypes.byref(_lib.ShardDesc(dims, 0, split + 1)), ctypes.byref(b0), None))
            b1 = _lib.ShardBufs(params=p1, wte=wte, tokens=t_dev, targets=g_dev, act_in=act, scratch=scratch,
                                scratch_bytes=need.value)
            ok(L.hy_shard_forward(d.h, ctypes.byref(_lib.ShardDesc(dims, split + 1, m.L + 2)), ctypes.byref(b1),
                                  ctypes.byref(loss)))
            assert abs(loss.value - loss_ref) / loss_ref < 1e-5
    finally:
        K.gemm_config(precision_fp32=False)
        d.close()
