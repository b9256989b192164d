"""ctypes binding of the C-ABI in include/hydra.h (libhydra.so, built in-tree by `make`).

The library is the product: there is no Python or CPU fallback. If it is missing or fails
to load, every entry point raises.
"""
import ctypes
import json
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhydra.so")

c_float_p = ctypes.POINTER(ctypes.c_float)

# name -> (restype, argtypes); mirrors include/hydra.h
_SIGS = {
    "hy_last_error": (ctypes.c_char_p, []),
    "hy_version": (ctypes.c_char_p, []),
    "hy_plan_json": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "hy_execute_json": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "hy_executor_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "hy_executor_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                       ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    "hy_executor_dump_params": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p]),
    "hy_executor_read_params": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.POINTER(ctypes.c_size_t)]),
    "hy_executor_destroy": (None, [ctypes.c_void_p]),
    "hy_kernel_launches": (ctypes.c_long, []),
    "hy_host_launch_us": (ctypes.c_double, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p]),
    "hy_gemm_config": (ctypes.c_int, [ctypes.c_int, ctypes.c_void_p, ctypes.c_long]),
    "hy_gemm": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_long,
                               ctypes.c_int, ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_void_p, ctypes.c_long,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_float, ctypes.c_int,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]),
    "hy_gemm_bf16": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_long, ctypes.c_int, ctypes.c_void_p, ctypes.c_long, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_long, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_long, ctypes.c_float, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_long]),
    "hy_to_bf16": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p]),
    "hy_layernorm_fwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 6),
    "hy_layernorm_bwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int] + [ctypes.c_void_p] * 6
                         + [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "hy_attention_fwd": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int] * 4 + [ctypes.c_void_p] * 3 + [ctypes.c_long]),
    "hy_attention_bwd": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int] * 4 + [ctypes.c_void_p] * 4 + [ctypes.c_long]),
    "hy_embed_fwd": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int] * 3 + [ctypes.c_void_p] * 4),
    "hy_embed_bwd": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int] * 4 + [ctypes.c_void_p] * 4),
    "hy_softmax_xent": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_long,
                                       ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p]),
    "hy_bias_grad": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_long,
                                    ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "hy_adam": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_void_p] * 4
                + [ctypes.c_float] * 5 + [ctypes.c_int]),
    "hy_adam_host_state": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_long] + [ctypes.c_void_p] * 5
                           + [ctypes.c_float] * 5 + [ctypes.c_int] * 3),
    "hy_flash_attention_fwd": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3),
    "hy_flash_attention_bwd": (ctypes.c_int, [ctypes.c_void_p] + [ctypes.c_int] * 3 + [ctypes.c_void_p] * 6),
    "hy_host_adam": (ctypes.c_int, [ctypes.c_long] + [ctypes.c_void_p] * 4 + [ctypes.c_float] * 5
                     + [ctypes.c_int] * 3),
    # device level (include/hydra.h "Device level")
    "hy_open": (ctypes.c_int, [ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "hy_close": (None, [ctypes.c_void_p]),
    "hy_lane_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "hy_arena_alloc": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "hy_arena_reset": (ctypes.c_int, [ctypes.c_void_p]),
    "hy_arena_peak": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]),
    "hy_pinned_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "hy_pinned_free": (ctypes.c_int, [ctypes.c_void_p]),
    "hy_copy_h2d": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "hy_copy_d2h": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t]),
    "hy_copy_p2p": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]),
    "hy_event_record": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "hy_lane_wait": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "hy_event_query": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]),
    "hy_event_elapsed": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_float)]),
    "hy_event_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "hy_lane_sync": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "hy_shard_scratch_bytes": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "hy_shard_forward": (ctypes.c_int, [ctypes.c_void_p] * 3 + [ctypes.POINTER(ctypes.c_double)]),
    "hy_shard_backward": (ctypes.c_int, [ctypes.c_void_p] * 3 + [ctypes.POINTER(ctypes.c_double)]),
}


class Dims(ctypes.Structure):  # hy_dims (include/hydra_gpt.h)
    _fields_ = [(n, ctypes.c_int) for n in ("V", "d", "L", "T", "B", "H")]


class ShardDesc(ctypes.Structure):  # hy_shard_desc
    _fields_ = [("dims", Dims), ("l0", ctypes.c_int), ("l1", ctypes.c_int)]


class ShardBufs(ctypes.Structure):  # hy_shard_bufs
    _fields_ = [(n, ctypes.c_void_p) for n in ("params", "wte", "tokens", "targets", "act_in", "act_out", "grad_in",
                                               "grad_out", "z_in", "z_out", "grads", "scratch")] + [
        ("scratch_bytes", ctypes.c_size_t)]

EXPORTED = sorted(_SIGS)

_lib = None


class HydraError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"hydra status {code}: {msg}")
        self.code = code


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `make` (or __graft_entry__.build())")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(code):
    if code != 0:
        raise HydraError(code, lib().hy_last_error().decode())
    return code


def call_json(fn_name, request: dict) -> dict:
    fn = getattr(lib(), fn_name)
    payload = json.dumps(request).encode()
    needed = ctypes.c_size_t(0)
    size = 1 << 20
    while True:
        buf = ctypes.create_string_buffer(size)
        rc = fn(payload, buf, size, ctypes.byref(needed))
        if rc == -9:  # HY_E_BUFFER_SMALL
            size = needed.value + 1
            continue
        check(rc)
        return json.loads(buf.value.decode())
