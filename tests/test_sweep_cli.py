"""`pascalsim sweep` as one device batch (pascal_sweep, cli.py) against the
reference CLI's sequential loop (proj/tools/pascalsim_cli.cpp:299-342) run on
the REAL reference library (oracle/_ref/libpascal_ref.so): every per-point
report file and sweep.csv must be byte-identical. Plus CPU checks of the CLI's
option handling (flag-over-file config resolution, gen presets)."""
import ctypes as C
import os
import subprocess
import sys

import pytest

import paper_2602_11530_b200 as pb
from paper_2602_11530_b200 import _lib, cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpascal_ref.so")


def ref():
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built (oracle/_ref)")
    return _lib.bind(C.CDLL(REF_SO), extensions=False)


def ref_sweep(trace_path, base, policies, fractions, out_dir):
    """The reference CLI's sweep loop, driven through the reference C ABI."""
    R = ref()
    os.makedirs(out_dir, exist_ok=True)
    t, p = C.c_void_p(), C.c_void_p()
    assert R.pascal_trace_load(trace_path.encode(), C.byref(t)) == 0
    assert R.pascal_profile_default(C.byref(p)) == 0
    rows = ["policy,capacity_fraction,slo_violation_rate,ttft_p50,ttft_p99,"
            "ttfat_attainment,throughput\n"]
    for pol in policies:
        for f in fractions:
            cfg = _lib.RunConfig()
            C.memmove(C.byref(cfg), C.byref(base), C.sizeof(cfg))
            cfg.policy = pol.encode()
            cfg.capacity_fraction = f
            prefix = f"{out_dir}/{pol}_f{f:.2f}"
            assert R.pascal_run(t, p, C.byref(cfg), prefix.encode(), None) == 0, \
                R.pascal_last_error()
            rep = C.c_void_p()
            assert R.pascal_report_load(prefix.encode(), C.byref(rep)) == 0
            vals = []
            for key in ("slo_violation_rate", "ttft_p50", "ttft_p99", "ttfat_attainment",
                        "throughput"):
                v = C.c_double()
                R.pascal_report_summary_value(rep, key.encode(), C.byref(v))
                vals.append(v.value)
            R.pascal_report_free(rep)
            rows.append(f"{pol},{f:.2f}," + ",".join(f"{v:.6f}" for v in vals) + "\n")
    with open(f"{out_dir}/sweep.csv", "w") as fh:
        fh.write("".join(rows))
    R.pascal_trace_free(t)
    R.pascal_profile_free(p)


def same_tree(a, b):
    fa, fb = sorted(os.listdir(a)), sorted(os.listdir(b))
    assert fa == fb
    for name in fa:
        assert open(os.path.join(a, name), "rb").read() == \
            open(os.path.join(b, name), "rb").read(), name


@pytest.mark.gpu
@pytest.mark.parametrize("instances,count,seed", [(1, 64, 1), (4, 300, 7)])
def test_sweep_matches_reference_cli_loop(tmp_path, instances, count, seed):
    trace = str(tmp_path / "t.csv")
    pb.Trace.preset("chat", count, 12.0, seed).save(trace)
    policies = ["fcfs", "rr", "oracle", "pascal"]
    fractions = [0.3, 0.5, 0.9]
    base = pb.run_config("pascal", instance_count=instances)
    ref_sweep(trace, base, policies, fractions, str(tmp_path / "ref"))
    rc = cli.main(["sweep", "--trace", trace, "--instances", str(instances), "--out-dir",
                   str(tmp_path / "gpu"), "--policies", *policies, "--capacity-fractions",
                   *map(str, fractions)])
    assert rc == 0
    same_tree(str(tmp_path / "ref"), str(tmp_path / "gpu"))


@pytest.mark.gpu
def test_sweep_ablation_flags_from_config_file(tmp_path):
    trace = str(tmp_path / "t.csv")
    pb.Trace.preset("mixed", 200, 8.0, 3, 0.25).save(trace)
    conf = tmp_path / "run.conf"
    conf.write_text("instance_count = 4\nno_migration = 1  # ablation\ntoken_quantum=300\n")
    base = pb.run_config("pascal", instance_count=4, no_migration=1, token_quantum=300)
    ref_sweep(trace, base, ["pascal"], [0.4, 0.6], str(tmp_path / "ref"))
    assert cli.main(["sweep", "--trace", trace, "--config", str(conf), "--out-dir",
                     str(tmp_path / "gpu"), "--policies", "pascal", "--capacity-fractions",
                     "0.4", "0.6"]) == 0
    same_tree(str(tmp_path / "ref"), str(tmp_path / "gpu"))


def test_config_resolution_flag_over_file(tmp_path):
    conf = tmp_path / "c.conf"
    conf.write_text("# comment\npolicy = rr\ninstance_count=3\ncapacity_fraction = 0.7\n"
                    "no_migration=1\npacer_slack_tokens = 4\nbogus\n")
    ap_args = ["run", "--trace", "x", "--config", str(conf), "--instances", "5"]
    import argparse
    p = argparse.ArgumentParser()
    cli.add_run_flags(p)
    p.add_argument("--out", default="report")
    p.add_argument("--events", default="")
    a = p.parse_args(ap_args[1:])
    o = cli.resolve(a)
    assert o["policy"] == "rr" and o["instances"] == 5 and o["capacity_fraction"] == 0.7
    assert o["no_migration"] is True and o["pacer_slack"] == 4 and o["quantum"] == 500


def test_gen_presets_match_reference_library(tmp_path):
    """`gen --preset chat|mixed|answering-char` writes the same trace file as
    the reference library's generator calls (cmd_gen)."""
    R = ref()
    for preset in ("chat", "mixed", "answering-char"):
        out = str(tmp_path / f"{preset}.csv")
        r = subprocess.run([sys.executable, "-m", "paper_2602_11530_b200", "gen", "--preset",
                            preset, "--count", "120", "--seed", "5", "--out", out],
                           capture_output=True, text=True, cwd=ROOT)
        assert r.returncode == 0, r.stderr
        assert r.stdout == f"wrote 120 requests to {out}\n"
        want = str(tmp_path / f"{preset}.ref.csv")
        if preset == "mixed":
            a, b, m = C.c_void_p(), C.c_void_p(), C.c_void_p()
            pc, pr, pa, _ = pb.PRESETS["chat"]
            hc, hr, ha, _ = pb.PRESETS["reasoning-heavy"]
            R.pascal_trace_generate(120, 12.0, pc.encode(), pr.encode(), pa.encode(), 5, 0,
                                    C.byref(a))
            R.pascal_trace_generate(120, 12.0, hc.encode(), hr.encode(), ha.encode(), 6, 0,
                                    C.byref(b))
            assert R.pascal_trace_mix(a, b, 0.5, 7, C.byref(m)) == 0
        else:
            m = C.c_void_p()
            pp, rr, aa, pre = pb.PRESETS[preset]
            R.pascal_trace_generate(120, 12.0, pp.encode(), rr.encode(), aa.encode(), 5,
                                    int(pre), C.byref(m))
        assert R.pascal_trace_save(m, want.encode()) == 0
        assert open(out, "rb").read() == open(want, "rb").read()


def test_sweep_without_a_device_fails_loudly(tmp_path):
    if pb.device_available():
        pytest.skip("a CUDA device is present")
    trace = str(tmp_path / "t.csv")
    pb.Trace.preset("chat", 16, 12.0, 1).save(trace)
    r = subprocess.run([sys.executable, "-m", "paper_2602_11530_b200", "sweep", "--trace", trace,
                        "--out-dir", str(tmp_path / "o")], capture_output=True, text=True,
                       cwd=ROOT)
    assert r.returncode == 1
    assert "pascalsim: sweep failed" in r.stderr
    assert not os.path.exists(tmp_path / "o" / "sweep.csv")
