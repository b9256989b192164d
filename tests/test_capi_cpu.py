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
