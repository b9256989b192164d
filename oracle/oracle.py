"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/liboracle_gpt.so
(CPU restatement of the shard numerics, see oracle/gpt_oracle.h), plus a pure-numpy
sharded-plan driver. Imported only by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline leg — never by the product path.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None


class Dims(ctypes.Structure):
    _fields_ = [("V", ctypes.c_int), ("d", ctypes.c_int), ("L", ctypes.c_int), ("T", ctypes.c_int),
                ("B", ctypes.c_int), ("H", ctypes.c_int)]


def make_dims(d, L, T, B, V=50257):
    return Dims(V, d, L, T, B, max(1, d // 64))


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(os.path.join(_HERE, "liboracle_gpt.so"))
        P = ctypes.c_void_p
        _lib.oracle_shard_fwd.argtypes = [P, P, ctypes.c_int, ctypes.c_int, P, P, P, P, P]
        _lib.oracle_shard_bwd.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, P, P, P, P, P]
        _lib.oracle_adam.argtypes = [ctypes.c_long, P, P, P, P] + [ctypes.c_float] * 5 + [ctypes.c_int]
        _lib.oracle_adam_state.argtypes = [ctypes.c_long, P, P, P, P] + [ctypes.c_float] * 5 + [ctypes.c_int] * 2
        _lib.oracle_train_step.argtypes = [P, P, P, P, ctypes.c_int, ctypes.c_float, P, P]
        _lib.oracle_train_step.restype = ctypes.c_double
        _lib.oracle_init_params.argtypes = [P, ctypes.c_uint64, P]
        _lib.oracle_make_tokens.argtypes = [P, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, P, P]
        _lib.oracle_threads.restype = ctypes.c_int
        _lib.oracle_set_bf16.argtypes = [ctypes.c_int]
    return _lib


def set_bf16(on):
    """Round the blocks' GEMM operands to bf16 (the GPU's "bf16" precision) in later calls."""
    lib().oracle_set_bf16(int(bool(on)))


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def total_floats(m):
    return layer_offset(m, m.L + 2)


def pad32(n):
    return (n + 31) // 32 * 32


def block_floats(d):
    sizes = [d, d, 3 * d * d, 3 * d, d * d, d, d, d, 4 * d * d, 4 * d, 4 * d * d, d]
    return sum(pad32(s) for s in sizes)


def layer_floats(m, layer):
    if layer == 0:
        return pad32(m.V * m.d) + pad32(m.T * m.d)
    if layer == m.L + 1:
        return 2 * pad32(m.d)
    return block_floats(m.d)


def layer_offset(m, layer):
    return sum(layer_floats(m, l) for l in range(layer))


def init_params(m, model_key):
    p = np.zeros(total_floats(m), dtype=np.float32)
    lib().oracle_init_params(ctypes.byref(m), ctypes.c_uint64(model_key), _p(p))
    return p


def tokens(m, seed, job, mb):
    tok = np.zeros(m.B * m.T, dtype=np.int32)
    tgt = np.zeros(m.B * m.T, dtype=np.int32)
    lib().oracle_make_tokens(ctypes.byref(m), ctypes.c_uint64(seed), job, mb, _p(tok), _p(tgt))
    return tok, tgt


def shard_fwd(m, params, l0, l1, tok, tgt, act_in):
    act_out = np.zeros(m.B * m.T * m.d, dtype=np.float32)
    loss = ctypes.c_double(0.0)
    lib().oracle_shard_fwd(ctypes.byref(m), _p(params), l0, l1, _p(tok), _p(tgt), _p(act_in), _p(act_out),
                           ctypes.byref(loss))
    return act_out, loss.value


def shard_bwd(m, params, grads, l0, l1, tok, tgt, act_in, grad_out):
    grad_in = np.zeros(m.B * m.T * m.d, dtype=np.float32)
    lib().oracle_shard_bwd(ctypes.byref(m), _p(params), _p(grads), l0, l1, _p(tok), _p(tgt), _p(act_in),
                           _p(grad_out), _p(grad_in))
    return grad_in


def adam(p, g, mom, var, lr, step, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0, bf16_state=False):
    lib().oracle_adam_state(p.size, _p(p), _p(g), _p(mom), _p(var), lr, beta1, beta2, eps, wd, step,
                            int(bf16_state))


def sharded_step(m, params, mom, var, starts, step, lr, tok, tgt, bf16_state=False):
    """One minibatch through the SHARP shard chain F(0..k-1), B(k-1..0), then Adam —
    the reference's task order (strategies.cpp:743-782). Returns the loss."""
    n_layers = m.L + 2
    bounds = list(starts) + [n_layers]
    k = len(starts)
    acts = [None] * k  # boundary activation out of shard s
    loss = None
    a = None
    for s in range(k):
        a_out, l = shard_fwd(m, params, bounds[s], bounds[s + 1], tok, tgt, a)
        if bounds[s + 1] == n_layers:
            loss = l
        acts[s] = a_out
        a = a_out
    grads = np.zeros_like(params)
    g = None
    for s in reversed(range(k)):
        ckpt = acts[s - 1] if s > 0 else None
        g = shard_bwd(m, params, grads, bounds[s], bounds[s + 1], tok, tgt, ckpt, g)
    adam(params, grads, mom, var, lr, step, bf16_state=bf16_state)
    return loss


M64 = (1 << 64) - 1


def mix64(x):
    """splitmix64 finalizer (include/hydra_gpt.h hy_mix64)."""
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def model_key(config_seed, model_index):
    """Init stream of config.models[model_index] (csrc/capi/execute.cpp exec_job_for)."""
    return mix64((config_seed * 0x100000001B3 + model_index) & M64)


def run_workload_cpu(config, shard_starts, max_minibatches=None, jobs=None, bf16_state=False):
    """Execute every job of a workload config on the CPU oracle in the SHARP chain order
    (per job: minibatches in order, each F(0..k-1), B(k-1..0), Adam). Returns
    (losses[job][mb], params[job])."""
    names = [m["name"] for m in config["models"]]
    seed = int(config.get("seed", 0))
    losses, params_out = {}, {}
    for j, job in enumerate(config["jobs"]):
        if jobs is not None and j not in jobs:
            continue
        mi = names.index(job["model"])
        g = config["models"][mi]["generator"]
        m = make_dims(d=g["d_model"], L=g["n_blocks"], T=g["seq_len"], B=g["batch_size"])
        p = init_params(m, model_key(seed, mi))
        mom, var = np.zeros_like(p), np.zeros_like(p)
        lr = float(job.get("hyperparams", {}).get("lr", "0.0001"))
        n_mb = job.get("epochs", 1) * job.get("minibatches_per_epoch", 1)
        if max_minibatches is not None:
            n_mb = min(n_mb, max_minibatches)
        ls = []
        for mb in range(n_mb):
            tok, tgt = tokens(m, seed, j, mb)
            ls.append(sharded_step(m, p, mom, var, shard_starts[j], mb + 1, lr, tok, tgt, bf16_state=bf16_state))
        losses[j], params_out[j] = ls, p
    return losses, params_out
