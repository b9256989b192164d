"""Runs the native host-library unit tests (tests/native/test_spillsim.cpp): the
reference's known-answer cases for the cost model, partitioner, virtual engine,
Sharded-LRTF, feasibility and config schema, against libhydra.so."""
import os
import subprocess

from conftest import ROOT


def test_native_known_answers():
    exe = os.path.join(ROOT, "build", "test_spillsim")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
