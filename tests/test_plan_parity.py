"""Bit-exact parity of the planning path against the REFERENCE.

tests/golden/plan_*.json were produced by oracle/_ref/plan_dump_ref — oracle/plan_dump.cpp
compiled against the reference sources in /root/reference/proj/core (oracle/Makefile).
The same driver compiled against this repo (build/plan_dump_b200) must reproduce them
byte-for-byte: partitions, ShardTask fields, LRTF estimates, dispatch order (task, device,
prefetch), every trace interval, the Chrome trace, RunReport JSON/CSV/text and the
canonical config serialization. Dispatch hashes also equal BASELINE.md §3.
"""
import json
import os
import subprocess

import pytest

from conftest import ROOT

CASES = sorted(f[:-5] for f in os.listdir(os.path.join(ROOT, "oracle", "cases")) if f.endswith(".json"))

BASELINE_HASHES = {  # BASELINE.md §3 (sharp, double buffering on), G = 1/2/4/8
    "c2": ["fc5367a99871a383", "a37bcffaaabca783", "25f45ee0a50e5183", "0a340c461eada783"],
    "c3": ["bdd31bb35dff9b83", "ba23da911c14ca83", "ab07a21619afec03", "0551683a70f42983"],
    "c4": ["579a1d73f8a85f83", "579a1d73f8a85f83"],
    "c5": ["4db0c8003926bb83", "4662d6ba9773a2a1", "59eca4aa2d44bf3d", "cf578b605fdf093d"],
}
BASELINE_MAKESPANS = {"c2": 1.4153651, "c3": 35.0099271, "c4": 6.4692646, "c5": 13.4574808}


def run_dump(case):
    exe = os.path.join(ROOT, "build", "plan_dump_b200")
    out = subprocess.run([exe, os.path.join(ROOT, "oracle", "cases", case + ".json")],
                         capture_output=True, text=True, check=True)
    return out.stdout


@pytest.mark.parametrize("case", CASES)
def test_plan_dump_byte_identical(case):
    mine = run_dump(case)
    with open(os.path.join(ROOT, "tests", "golden", f"plan_{case}.json")) as f:
        golden = f.read()
    if mine != golden:
        a, b = json.loads(mine), json.loads(golden)
        for ra, rb in zip(a.get("runs", []), b.get("runs", [])):
            for k in rb:
                assert ra.get(k) == rb[k], f"{case} {rb['strategy']} G={rb['gpus']} db={rb['double_buffering']}: {k}"
        assert a == b
    assert mine == golden


@pytest.mark.parametrize("case", sorted(BASELINE_HASHES))
def test_dispatch_hash_matches_baseline_md(case):
    with open(os.path.join(ROOT, "tests", "golden", f"plan_{case}.json")) as f:
        runs = json.load(f)["runs"]
    got = [r["dispatch_hash"] for r in runs if r["strategy"] == "sharp" and r["double_buffering"]]
    assert got == BASELINE_HASHES[case]
    g1 = [r for r in runs if r["strategy"] == "sharp" and r["double_buffering"] and r["gpus"] == 1][0]
    assert abs(float(g1["makespan"]) - BASELINE_MAKESPANS[case]) < 1e-6


def test_sharp_jobs_pinned_to_one_device_with_double_buffering():
    """with DB on every job stays on the device it first lands on."""
    with open(os.path.join(ROOT, "tests", "golden", "plan_c3.json")) as f:
        runs = json.load(f)["runs"]
    for r in runs:
        if r["strategy"] != "sharp":
            continue
        tasks = r["tasks"]
        devs = {}
        for t, d, _ in r["dispatch"]:
            devs.setdefault(tasks[t][0], set()).add(d)
        if r["double_buffering"]:
            assert all(len(v) == 1 for v in devs.values())
