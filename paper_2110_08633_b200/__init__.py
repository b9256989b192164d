"""B200-native shard-execution path of Hydra (arXiv 2110.08633).

Native library: paper_2110_08633_b200/libhydra.so (C++ planner + sm_100a kernels + C-ABI,
include/hydra.h). Python here is only a thin ctypes layer.
"""
from ._lib import HydraError, call_json, lib  # noqa: F401

__all__ = ["HydraError", "call_json", "lib", "plan", "execute"]


def plan(config: dict, strategy: str = "sharp", gpus: int = 0, double_buffering=None, trace=False) -> dict:
    req = {"config": config, "strategy": strategy, "gpus": gpus, "trace": trace}
    if double_buffering is not None:
        req["double_buffering"] = double_buffering
    return call_json("hy_plan_json", req)


def execute(config: dict, **kw) -> dict:
    req = {"config": config}
    req.update(kw)
    return call_json("hy_execute_json", req)


class Executor:
    """Stateful B200 executor over the C-ABI (hy_executor_*): setup once, run passes."""

    def __init__(self, config: dict, **kw):
        import ctypes
        import json as _json

        from ._lib import check

        req = {"config": config}
        req.update(kw)
        h = ctypes.c_void_p()
        check(lib().hy_executor_create(_json.dumps(req).encode(), ctypes.byref(h)))
        self._h = h

    def run(self, passes: int, timed: bool = True, trace: bool = False, interval_log: bool = False) -> dict:
        """Replay the plan `passes` times (hy_executor_run). interval_log: timed passes also log
        every compute op and host<->device copy (result "links": copy-only link time and the
        transfer-overlap fraction per GPU) — measure throughput on passes without it."""
        import ctypes
        import json as _json

        from ._lib import check

        size = 1 << 22
        needed = ctypes.c_size_t(0)
        while True:
            buf = ctypes.create_string_buffer(size)
            mode = (2 if interval_log else 1) if timed else 0
            rc = lib().hy_executor_run(self._h, int(passes), mode, int(trace), buf, size, ctypes.byref(needed))
            if rc == -9:
                size = needed.value + 1
                continue
            check(rc)
            return _json.loads(buf.value.decode())

    def dump_params(self, directory: str):
        from ._lib import check

        check(lib().hy_executor_dump_params(self._h, directory.encode()))

    def read_params(self, job: int):
        """Job `job`'s host parameter vector (final after a pass) as a float32 numpy array."""
        import ctypes

        import numpy as np

        from ._lib import check

        n = ctypes.c_size_t(0)
        check(lib().hy_executor_read_params(self._h, int(job), None, 0, ctypes.byref(n)))
        out = np.empty(n.value, dtype=np.float32)
        check(lib().hy_executor_read_params(self._h, int(job), out.ctypes.data_as(ctypes.c_void_p), out.size,
                                            ctypes.byref(n)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().hy_executor_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def kernel_launches() -> int:
    return int(lib().hy_kernel_launches())
