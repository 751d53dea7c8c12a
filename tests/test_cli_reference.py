"""The reference's command-line tool (proj/tools/gridadmm.cpp), compiled
UNCHANGED twice — against libgridadmm.so and against the reference library
(oracle/Makefile targets _ref/gridadmm_cli and _ref/gridadmm_cli_ref, with
tests/c/CLI11.hpp standing in for the CLI11 header) — run on the same
inputs: identical exit codes, stdout, error messages, and output files byte
for byte except the wall-clock fields (SURVEY.md §8(b) "Callers").  Input
errors run on CPU; solves need the GPU."""
import os
import re
import subprocess

import pytest

from conftest import REPO, case_path

CLI = os.path.join(REPO, "oracle", "_ref", "gridadmm_cli")
CLI_REF = os.path.join(REPO, "oracle", "_ref", "gridadmm_cli_ref")


def run(exe, *args):
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    return subprocess.run([exe, *args], capture_output=True, text=True, timeout=600)


def mask(name, text):
    if name == "solution.json":
        return re.sub(r'("phase_times_s": \{)[^}]*(\})', r"\1\2", text)
    rows = [ln.split(",") for ln in text.strip("\n").split("\n")]
    col = {"convergence.csv": "elapsed_s", "periods.csv": "time_s"}[name]
    k = rows[0].index(col)
    return "\n".join(",".join(r[:k] + r[k + 1:]) for r in rows)


@pytest.mark.parametrize("args", [
    ["solve"],                                   # missing --case
    ["solve", "--case", "/no/such/case.m"],      # unreadable case
    ["solve", "--case", case_path("case9"), "--preset", "case_unknown"],
    ["solve", "--case", case_path("case9"), "--beta0", "0"],
    ["solve", "--case", case_path("case9"), "--max-outer", "0"],
    ["track", "--case", case_path("case9")],     # missing --profile
    ["bogus"],
])
def test_cli_input_errors_match_reference(args):
    a, b = run(CLI, *args), run(CLI_REF, *args)
    assert a.returncode == b.returncode != 0
    assert a.stdout == b.stdout and a.stderr == b.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("cmd,extra", [
    ("solve", ["--preset", "case9", "--eps", "1e-4", "--ref-objective", "5296.69"]),
    ("solve", ["--preset", "case9", "--max-outer", "1", "--max-inner", "40"]),   # exit code 2
    ("track", ["--preset", "case9", "--eps", "1e-4"]),
])
def test_cli_runs_match_reference(tmp_path, cmd, extra):
    args = [cmd, "--case", case_path("case9"), *extra]
    if cmd == "track":
        prof = tmp_path / "profile.csv"
        prof.write_text("period,multiplier\n1,1.0\n2,1.005\n3,1.0\n")
        args += ["--profile", str(prof)]
    outs = {}
    for tag, exe in (("mine", CLI), ("ref", CLI_REF)):
        d = tmp_path / tag
        r = run(exe, *args, "--out-dir", str(d))
        outs[tag] = (r, d)
    (a, da), (b, db) = outs["mine"], outs["ref"]
    assert a.returncode == b.returncode, (a.stderr, b.stderr)
    assert a.stdout == b.stdout and a.stderr == b.stderr
    files = sorted(os.listdir(db))
    assert files == sorted(os.listdir(da)) and files
    for f in files:
        assert mask(f, (da / f).read_text()) == mask(f, (db / f).read_text()), f
