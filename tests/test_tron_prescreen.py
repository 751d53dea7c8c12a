"""The Cauchy backtracking pre-screen (tron.cuh cauchy_skip) skips only
trials whose failure it proves, so the step is bit-identical to the
reference's loop (proj/src/tron.cpp:101-137).  Host check (no GPU): the
product's cauchy_point is compiled with g++ -ffp-contract=off (the same IEEE
operations as the -fmad=false device build) and compared bit for bit with
the reference loop on random and adversarial instances (tests/c/
cauchy_skip_check.cpp); the GPU side is covered by the TRON-core and
residual-series parity tests."""
import os
import subprocess

from conftest import REPO


def test_cauchy_prescreen_is_exact(tmp_path):
    exe = tmp_path / "csc"
    src = os.path.join(REPO, "tests", "c", "cauchy_skip_check.cpp")
    inc = os.path.join(REPO, "paper_2110_06879_b200", "csrc")
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-I", inc,
                        src, "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe), "300000", "11"], capture_output=True, text=True, timeout=600)
    bad, skipped, trials = (int(v) for v in out.stdout.split())
    assert bad == 0, out.stdout
    assert skipped > 0.1 * trials  # the screen does skip work on these instances
