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
