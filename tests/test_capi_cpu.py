"""CPU-side checks of the C-ABI boundary: the library loads without a GPU, exports every
symbol include/hydra.h declares, maps reference exceptions to status codes, and the JSON
planning entry reproduces the reference goldens."""
import json
import os
import re

import pytest

from conftest import ROOT

import paper_2110_08633_b200 as P
from paper_2110_08633_b200 import _lib


def declared_symbols():
    with open(os.path.join(ROOT, "include", "hydra.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(hy_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 20
    lib = P.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTED) == syms  # the Python binding covers exactly the header


def test_version_and_error_text():
    assert b"sm_100a" in P.lib().hy_version()
    with pytest.raises(P.HydraError) as e:
        P.plan({"schema_version": 1})
    assert e.value.code == -2  # ConfigError
    assert "missing field" in str(e.value)


def test_error_codes_map_reference_exceptions():
    with open(os.path.join(ROOT, "configs", "c1_tiny.json")) as f:
        cfg = json.load(f)
    cfg["cluster"]["devices"][0]["mem_bytes"] = 1e6  # embedding alone exceeds the cap
    with pytest.raises(P.HydraError) as e:
        P.plan(cfg)
    assert e.value.code == -5  # SingleLayerTooLarge -> HY_E_INFEASIBLE
    with pytest.raises(P.HydraError) as e:
        P.plan(cfg, strategy="pipeline-parallel")
    assert e.value.code in (-1, -5)


@pytest.mark.parametrize("case,hash_g1", [("c2_gpt2small_x8", "fc5367a99871a383"), ("c3_gpt2xl_x16", "bdd31bb35dff9b83")])
def test_plan_json_matches_reference(case, hash_g1):
    with open(os.path.join(ROOT, "configs", case + ".json")) as f:
        cfg = json.load(f)
    r = P.plan(cfg, gpus=1)
    assert r["dispatch_hash"] == hash_g1
    with open(os.path.join(ROOT, "tests", "golden", "plan_" + case.split("_")[0] + ".json")) as f:
        gold = [x for x in json.load(f)["runs"] if x["strategy"] == "sharp" and x["gpus"] == 1
                and x["double_buffering"]][0]
    assert [p["shard_starts"] for p in r["partitions"]] == [p["shard_starts"] for p in gold["partitions"]]
    assert [[d[0], d[1]] for d in r["dispatch"]] == [[d[0], d[1]] for d in gold["dispatch"]]
    assert abs(r["makespan_s"] - float(gold["makespan"])) == 0.0


@pytest.mark.parametrize("bf16", [False, True])
def test_host_adam_matches_oracle(bf16):
    """Host-side AdamW (the executor's host_opt_fraction path) against the
    CPU oracle's update over 3 steps; bf16 moments round RNE like the oracle's emulation."""
    import numpy as np
    from oracle import oracle as O

    rng = np.random.default_rng(7)
    n = 100_003  # ragged: not a multiple of the vector width or the thread split
    p0 = rng.standard_normal(n).astype(np.float32) * 0.02
    po, mo, vo = p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    ph = p0.copy()
    mh = np.zeros(n, np.uint16 if bf16 else np.float32)
    vh = np.zeros_like(mh)
    for step in (1, 2, 3):
        g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
        g[::97] = 0.0
        O.adam(po, g, mo, vo, 3e-4, step, wd=0.01, bf16_state=bf16)
        rc = P.lib().hy_host_adam(n, ph.ctypes.data, g.ctypes.data, mh.ctypes.data, vh.ctypes.data, 3e-4, 0.9,
                                  0.999, 1e-8, 0.01, step, int(bf16), 3)
        assert rc == 0
    as_f = (lambda a: (a.astype(np.uint32) << 16).view(np.float32)) if bf16 else (lambda a: a)
    # identical formula; only FMA contraction may differ -> a few ulp
    np.testing.assert_allclose(ph, po, rtol=2e-6, atol=1e-9)
    np.testing.assert_allclose(as_f(mh), mo, rtol=1e-2 if bf16 else 2e-6, atol=1e-9)
    np.testing.assert_allclose(as_f(vh), vo, rtol=1e-2 if bf16 else 2e-6, atol=1e-12)
    assert P.lib().hy_host_adam(-1, 0, 0, 0, 0, 1e-3, 0.9, 0.999, 1e-8, 0.0, 1, 0, 1) == -1


@pytest.mark.parametrize("field,value,msg", [("schedule", "eager", "schedule must be"),
                                             ("precision", "fp16", "precision must be"),
                                             ("opt_state", "fp8", "opt_state must be"),
                                             ("host_opt_fraction", 1.5, "host_opt_fraction")])
def test_execute_request_validation_without_gpu(field, value, msg):
    """Execution-request fields are validated before any device work, so a bad request fails
    with InvalidArgument (HY_E_INVALID, -1) and the reason even on a host without a GPU."""
    with open(os.path.join(ROOT, "configs", "c1_tiny.json")) as f:
        cfg = json.load(f)
    with pytest.raises(P.HydraError) as e:
        P.execute(cfg, **{field: value})
    assert e.value.code == -1 and msg in str(e.value), (e.value.code, str(e.value))


def test_pinned_shard_boundaries():
    """Boundary reuse (partitioner.cpp:157-231) through the request: a list of starts or the
    boundary text of boundaries_to_text; validated against the cap like the reference does."""
    with open(os.path.join(ROOT, "configs", "c3_gpt2xl_x16.json")) as f:
        cfg = json.load(f)
    model = dict(cfg["models"][0])
    model["generator"] = dict(model["generator"], batch_size=2)
    cfg["models"] = [model]
    cfg["jobs"] = [dict(cfg["jobs"][0], batch_size=2, minibatches_per_epoch=2)]
    assert P.plan(cfg)["partitions"][0]["shard_starts"] == [0]  # b2 fits the 24e9 cap whole
    cfg["options"] = dict(cfg["options"], buffer_policy={"kind": "absolute", "value": 5359724800.0})
    for pin in ([0, 24, 48], "0\n24\n48\n"):
        r = P.call_json("hy_plan_json", {"config": cfg, "shard_boundaries": [pin]})
        assert r["partitions"][0]["shard_starts"] == [0, 24, 48]
        assert len(r["tasks"]) == 2 * 2 * 3  # minibatches x (F + B) x shards
    with pytest.raises(P.HydraError) as e:  # not strictly increasing
        P.call_json("hy_plan_json", {"config": cfg, "shard_boundaries": [[0, 24, 24]]})
    assert e.value.code == -1 and "strictly increasing" in str(e.value)
    with pytest.raises(P.HydraError):  # only SHARP partitions spilled shards
        P.call_json("hy_plan_json", {"config": cfg, "strategy": "task-parallel", "shard_boundaries": [[0, 24]]})
