"""C-ABI checks that need no GPU: symbol set, status codes and error messages
(mirroring proj/tests/test_capi.cpp), host-side file formats byte-identical to
the reference library (oracle/_ref/libpascal_ref.so, when built here), and the
no-CPU-fallback rule (a run without a CUDA device fails loudly)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2602_11530_b200 as pb
from paper_2602_11530_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libpascal_ref.so")


def lib():
    return _lib.load()


def ref():
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built (oracle/_ref)")
    return _lib.bind(C.CDLL(REF_SO), extensions=False)


def test_exports_every_declared_symbol_and_nothing_else():
    declared = set()
    for h in ("pascal.h", "pascal_b200.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        declared |= set(re.findall(r"\b(pascal_[a-z0-9_]+)\s*\(", text))
    assert declared == set(_lib.ABI_SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], check=True,
                         capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert exported == declared
    L = lib()
    for s in declared:
        assert hasattr(L, s)


def test_reference_19_symbols_are_a_subset():
    if not os.path.exists(REF_SO):
        pytest.skip("reference library not built")
    out = subprocess.run(["nm", "-D", "--defined-only", REF_SO], check=True,
                         capture_output=True, text=True).stdout
    ref_c = {ln.split()[-1] for ln in out.splitlines()
             if " T pascal_" in ln}
    assert len(ref_c) == 19
    assert ref_c <= set(_lib.ABI_SYMBOLS)


def test_trace_generate_save_load(tmp_path):
    t = pb.Trace.generate(50, 10.0, "constant:64", "uniform:0:200", "uniform:1:50", 123)
    assert len(t) == 50
    p = str(tmp_path / "t.csv")
    t.save(p)
    back = pb.Trace.load(p)
    assert len(back) == 50


def test_error_reporting_carries_a_message():
    L = lib()
    out = C.c_void_p()
    assert L.pascal_trace_generate(10, -1.0, b"constant:64", b"constant:0", b"constant:1", 0, 0,
                                   C.byref(out)) == _lib.INVALID_ARGUMENT
    assert len(L.pascal_last_error()) > 0
    assert L.pascal_trace_load(b"/nonexistent/path.csv", C.byref(out)) == _lib.IO
    assert L.pascal_trace_generate(10, 1.0, b"bogus:1", b"constant:0", b"constant:1", 0, 0,
                                   C.byref(out)) == _lib.INVALID_ARGUMENT
    assert L.pascal_trace_load(None, C.byref(out)) == _lib.INVALID_ARGUMENT
    assert L.pascal_last_error() == b"null argument"
    assert L.pascal_trace_save(None, b"x") == _lib.INVALID_ARGUMENT
    prof = C.c_void_p()
    assert L.pascal_profile_default(C.byref(prof)) == _lib.OK
    assert L.pascal_last_error() == b""  # success clears the error
    L.pascal_profile_free(prof)
    assert L.pascal_trace_size(None) == 0
    L.pascal_trace_free(None)
    L.pascal_profile_free(None)
    L.pascal_report_free(None)
    L.pascal_run_config_init(None)


def test_profile_manipulation(tmp_path):
    p = pb.Profile.default()
    p.set("decode_base", 0.02)
    with pytest.raises(pb.PascalError) as e:
        p.set("not_a_field", 1.0)
    assert e.value.status == _lib.INVALID_ARGUMENT
    path = str(tmp_path / "p.txt")
    p.save(path)
    pb.Profile.load(path)
    (tmp_path / "bad.txt").write_text("not-a-profile\n")
    with pytest.raises(pb.PascalError) as e:
        pb.Profile.load(str(tmp_path / "bad.txt"))
    assert e.value.status == _lib.IO
    (tmp_path / "neg.txt").write_text("pascal-profile-v1\ndecode_base=-1\n")
    with pytest.raises(pb.PascalError) as e:
        pb.Profile.load(str(tmp_path / "neg.txt"))
    assert e.value.status == _lib.INVALID_ARGUMENT


def test_calibration_recovers_a_plane(tmp_path):
    s = tmp_path / "calib.csv"
    s.write_text("".join(f"{b},{kv},{0.01 + 0.002 * b + 1e-6 * kv!r}\n"
                         for b in (1, 4, 16) for kv in (100, 1000, 10000)))
    p = pb.Profile.default()
    assert p.calibrate(str(s)) < 1e-9
    (tmp_path / "few.csv").write_text("1,2,0.1\n")
    with pytest.raises(pb.PascalError) as e:
        p.calibrate(str(tmp_path / "few.csv"))
    assert e.value.status == _lib.INVALID_ARGUMENT


def test_run_config_defaults_and_bad_policy():
    cfg = pb.run_config()
    assert (cfg.instance_count, cfg.token_quantum, cfg.demotion_threshold) == (8, 500, 5000)
    assert cfg.policy == b"pascal" and cfg.target_tpot == 0.1 and cfg.qoe_threshold == 0.95
    t = pb.Trace.generate(5, 10.0, "constant:64", "uniform:0:20", "uniform:1:4", 7)
    with pytest.raises(pb.PascalError) as e:
        pb.run(t, pb.Profile.default(), pb.run_config("nope"), "/tmp/x")
    assert e.value.status == _lib.INVALID_ARGUMENT
    assert "unknown policy" in e.value.message


def test_no_cpu_fallback_without_a_device(tmp_path):
    if pb.device_available():
        pytest.skip("a CUDA device is present")
    t = pb.Trace.generate(5, 10.0, "constant:64", "uniform:0:20", "uniform:1:4", 7)
    with pytest.raises(pb.PascalError) as e:
        pb.run(t, pb.Profile.default(), pb.run_config(instance_count=2,
                                                       capacity_fraction=0.5),
               str(tmp_path / "r"))
    assert e.value.status == _lib.INTERNAL
    assert "CUDA" in e.value.message


# ---------------------------------------------------------- byte parity vs reference
def _ref_trace(R, *gen):
    out = C.c_void_p()
    assert R.pascal_trace_generate(*gen, C.byref(out)) == 0
    return out


GENS = [
    (300, 12.0, b"uniform:64:512",
     b"hist:256=0.35,512=0.30,768=0.20,1024=0.10,1536=0.04,2048=0.01", b"uniform:256:1024",
     1, 0),
    (50, 3.5, b"constant:64", b"uniform:0:200", b"uniform:1:50", 123, 1),
]


@pytest.mark.parametrize("gen", GENS)
def test_trace_text_file_byte_identical_to_reference(gen, tmp_path):
    R = ref()
    rt = _ref_trace(R, *gen)
    a, b = str(tmp_path / "ref.csv"), str(tmp_path / "mine.csv")
    assert R.pascal_trace_save(rt, a.encode()) == 0
    n, rate, pd, rd, ad, seed, pre = gen
    pb.Trace.generate(n, rate, pd.decode(), rd.decode(), ad.decode(), seed, bool(pre)).save(b)
    assert open(a, "rb").read() == open(b, "rb").read()
    # and loading the reference's file gives the same file back
    pb.Trace.load(a).save(b)
    assert open(a, "rb").read() == open(b, "rb").read()
    R.pascal_trace_free(rt)


def test_mix_byte_identical_to_reference(tmp_path):
    R = ref()
    a = _ref_trace(R, *GENS[0])
    b = _ref_trace(R, 300, 12.0, b"uniform:64:512", b"uniform:2048:8192", b"uniform:128:512",
                   2, 0)
    m = C.c_void_p()
    assert R.pascal_trace_mix(a, b, 0.25, 3, C.byref(m)) == 0
    pa, pm = str(tmp_path / "ref.csv"), str(tmp_path / "mine.csv")
    R.pascal_trace_save(m, pa.encode())
    pb.Trace.preset("mixed", 300, 12.0, 1).save(pm)
    assert open(pa, "rb").read() == open(pm, "rb").read()


def test_profile_file_and_calibration_identical_to_reference(tmp_path):
    R = ref()
    rp = C.c_void_p()
    R.pascal_profile_default(C.byref(rp))
    mine = pb.Profile.default()
    for k, v in (("decode_base", 0.0123456789), ("swap_bandwidth", float("inf")),
                 ("fabric_latency", 1e-7)):
        R.pascal_profile_set(rp, k.encode(), v)
        mine.set(k, v)
    s = tmp_path / "s.csv"
    s.write_text("# batch,kv,seconds\n" + "".join(
        f"{b},{kv},{0.02 + 0.0015 * b + 2e-6 * kv + ((b * 7 + kv) % 5) * 1e-4!r}\n"
        for b in (1, 2, 4, 8, 16, 32) for kv in (100, 1000, 10000, 50000)))
    r1, r2 = C.c_double(), C.c_double()
    assert R.pascal_profile_calibrate(str(s).encode(), rp, C.byref(r1)) == 0
    r2 = mine.calibrate(str(s))
    assert r1.value == r2
    a, b = str(tmp_path / "a.txt"), str(tmp_path / "b.txt")
    R.pascal_profile_save(rp, a.encode())
    mine.save(b)
    assert open(a, "rb").read() == open(b, "rb").read()


def test_report_load_and_compare_identical_to_reference(tmp_path):
    """Reports written by the reference are loaded/compared identically by ours."""
    R = ref()
    t = _ref_trace(R, 120, 10.0, b"uniform:64:512", b"uniform:0:900", b"uniform:16:400", 5, 0)
    prof = C.c_void_p()
    R.pascal_profile_default(C.byref(prof))
    R.pascal_profile_set(prof, b"decode_base", 0.005)
    prefixes = []
    for pol in (b"fcfs", b"pascal"):
        cfg = _lib.RunConfig()
        R.pascal_run_config_init(C.byref(cfg))
        cfg.policy = pol
        cfg.instance_count = 2
        cfg.capacity_fraction = 0.5
        p = str(tmp_path / pol.decode())
        assert R.pascal_run(t, prof, C.byref(cfg), p.encode(), None) == 0
        prefixes.append(p)
    names = ["fcfs", "pascal"]
    PP = C.c_char_p * 2
    ra, rb = str(tmp_path / "ref_cmp.txt"), str(tmp_path / "mine_cmp.txt")
    assert R.pascal_compare(PP(*[p.encode() for p in prefixes]), PP(b"fcfs", b"pascal"), 2,
                            ra.encode()) == 0
    pb.compare(prefixes, names, rb)
    assert open(ra, "rb").read() == open(rb, "rb").read()
    rep = pb.Report.load(prefixes[1])
    v = C.c_double()
    rr = C.c_void_p()
    assert R.pascal_report_load(prefixes[1].encode(), C.byref(rr)) == 0
    for key in ("ttft_mean", "ttft_p50", "ttft_p90", "ttft_p95", "ttft_p99",
                "slo_violation_rate", "ttfat_attainment", "throughput"):
        R.pascal_report_summary_value(rr, key.encode(), C.byref(v))
        assert rep.summary_value(key) == v.value
    with pytest.raises(pb.PascalError) as e:
        rep.summary_value("banana")
    assert e.value.status == _lib.INVALID_ARGUMENT
    with pytest.raises(pb.PascalError) as e:
        pb.compare(prefixes[:1], names[:1], rb)
    assert e.value.status == _lib.INVALID_ARGUMENT
