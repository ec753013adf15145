"""The reference's own C-ABI callers, compiled unmodified from
/root/reference/proj against libpascal.so (oracle/Makefile `callers`;
INTEGRATION.md §2): proj/tests/test_capi.cpp with the doctest shim and the CLI
proj/tools/pascalsim_cli.cpp with the CLI11 shim (tests/shim/). Each is also
linked to the reference library itself, which pins the shims; the CLI's
outputs through libpascal.so must be byte-identical to the reference's."""
from __future__ import annotations

import filecmp
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
BIN = {k: os.path.join(REF, k) for k in ("test_capi_ref", "test_capi_b200", "pascalsim_ref",
                                          "pascalsim_b200")}


def need(*names):
    for n in names:
        if not os.path.exists(BIN[n]):
            pytest.skip(f"{n} not built (oracle/Makefile callers needs /root/reference)")


def run(args, cwd, **kw):
    p = subprocess.run(args, cwd=cwd, capture_output=True, text=True, timeout=600, **kw)
    assert p.returncode == 0, (args, p.stdout[-2000:], p.stderr[-2000:])
    return p.stdout


def test_reference_capi_test_passes_on_reference_library(tmp_path):
    need("test_capi_ref")
    out = run([BIN["test_capi_ref"]], str(tmp_path), env={**os.environ, "TMPDIR": str(tmp_path)})
    assert "| 0 failed" in out


def test_cli_gen_is_byte_identical_host_only(tmp_path):
    """`pascalsim gen` (trace generation + mixing) is host code in both
    libraries: identical files, no GPU needed."""
    need("pascalsim_ref", "pascalsim_b200")
    for tag in ("ref", "b200"):
        d = tmp_path / tag
        d.mkdir()
        run([BIN["pascalsim_" + tag], "gen", "--preset", "chat", "--count", "300", "--rate", "12",
             "--seed", "7", "--out", "a.csv"], str(d))
        run([BIN["pascalsim_" + tag], "gen", "--preset", "reasoning-heavy", "--count", "300",
             "--rate", "12", "--seed", "8", "--out", "b.csv"], str(d))
        run([BIN["pascalsim_" + tag], "gen", "--preset", "chat", "--count", "300", "--rate", "12",
             "--seed", "7", "--mix-trace", "b.csv", "--mix-fraction", "0.25", "--out", "m.csv"],
            str(d))
    for f in ("a.csv", "b.csv", "m.csv"):
        assert filecmp.cmp(tmp_path / "ref" / f, tmp_path / "b200" / f, shallow=False), f


@pytest.mark.gpu
def test_reference_capi_test_passes_on_libpascal(tmp_path):
    need("test_capi_b200")
    out = run([BIN["test_capi_b200"]], str(tmp_path), env={**os.environ, "TMPDIR": str(tmp_path)})
    assert "| 0 failed" in out


@pytest.mark.gpu
def test_reference_cli_relinked_is_byte_identical(tmp_path):
    """gen -> run (report + event log) -> sweep -> compare through the
    unmodified reference CLI: libpascal.so (GPU) vs the reference library."""
    need("pascalsim_ref", "pascalsim_b200")
    for tag in ("ref", "b200"):
        d = tmp_path / tag
        d.mkdir()
        exe = BIN["pascalsim_" + tag]
        run([exe, "gen", "--preset", "chat", "--count", "400", "--rate", "12", "--seed", "1",
             "--out", "t.csv"], str(d))
        with open(d / "run.cfg", "w") as f:
            f.write("instances = 4  # config file, flags override\ncapacity_fraction = 0.3\n"
                    "policy = fcfs\n")
        run([exe, "run", "--trace", "t.csv", "--config", "run.cfg", "--policy", "pascal",
             "--out", "rep", "--events", "ev.log"], str(d))
        run([exe, "run", "--trace", "t.csv", "--instances", "2", "--capacity-fraction", "0.5",
             "--policy", "pascal", "--non-adaptive", "--out", "na"], str(d))
        run([exe, "sweep", "--trace", "t.csv", "--instances", "2", "--policies", "fcfs", "rr",
             "oracle", "pascal", "--capacity-fractions", "0.3", "0.6", "--out-dir", "sw"],
            str(d))
        run([exe, "compare", "--reports", "sw/fcfs_f0.30", "sw/pascal_f0.30", "rep",
             "--names", "fcfs", "pascal", "c2", "--out", "cmp.txt"], str(d))
    files = ["t.csv", "ev.log", "cmp.txt", "sw/sweep.csv"]
    for p in ("rep", "na", "sw/fcfs_f0.30", "sw/rr_f0.60", "sw/oracle_f0.30", "sw/pascal_f0.60"):
        files += [f"{p}.requests.csv", f"{p}.summary.txt", f"{p}.bins.csv"]
    for f in files:
        assert filecmp.cmp(tmp_path / "ref" / f, tmp_path / "b200" / f, shallow=False), f
