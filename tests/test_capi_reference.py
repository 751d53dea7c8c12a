"""The reference's own C-ABI test, proj/tests/test_capi.cpp, compiled
UNCHANGED against libgridadmm.so (oracle/Makefile target _ref/test_capi, with
tests/c/doctest.h standing in for the doctest header): the drop-in proof of
SURVEY.md §8(b) "Callers".  The host-only cases run here; the solve and
tracking cases need the GPU."""
import os
import subprocess

import pytest

from conftest import REPO

EXE = os.path.join(REPO, "oracle", "_ref", "test_capi")


def run(*args):
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/test_capi not built (needs /root/reference at build time)")
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("case", ["network load, dimensions and errors",
                                  "config: set, get, validation, presets"])
def test_reference_capi_host_cases(case):
    r = run(f"--tc={case}")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[pass] " + case in r.stdout


@pytest.mark.gpu
def test_reference_capi_all_cases():
    r = run()
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 5 run, 0 failed" in r.stdout, r.stdout
