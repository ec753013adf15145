"""The C restatement (oracle/pascal_oracle.c) is pinned against the REAL
reference: its records and decision logs must hash to the goldens produced by
oracle/make_golden.py from /root/reference (CPU only)."""
import os
import subprocess

import pytest

from cases import BY_NAME, CASES, cfg_text
from harness import ORACLE_DUMP, build_trace, golden, sha_file

GOLD = golden()
FAST = [c for c in CASES if c["name"] in GOLD and c["size"] in ("tiny", "small")]
FAST += [BY_NAME[n] for n in ("mix500_pascal", "c5_s7_k6_pascal", "c5_s7_k6_nonadaptive",
                              "wide40_pascal") if n in GOLD]


@pytest.mark.parametrize("c", FAST, ids=[c["name"] for c in FAST])
def test_oracle_matches_reference(c, tmp_path):
    if not os.path.exists(ORACLE_DUMP):
        pytest.skip("oracle/_build/oracle_dump not built")
    g = GOLD[c["name"]]
    t = build_trace(c["trace"])
    hexp = str(tmp_path / "t.hex")
    t.save_hex(hexp)
    assert sha_file(hexp) == g["trace"], "host trace generator diverges from the reference"
    cfgp = tmp_path / "cfg"
    cfgp.write_text(cfg_text(c))
    rec, ev = str(tmp_path / "o.rec"), str(tmp_path / "o.ev")
    subprocess.run([ORACLE_DUMP, "run", hexp, str(cfgp), rec, ev], check=True, timeout=300)
    assert sha_file(rec) == g["records"]
    assert sha_file(ev) == g["events"]
    cap = subprocess.run([ORACLE_DUMP, "capacity", hexp, str(cfgp)], check=True,
                         capture_output=True, text=True).stdout.strip()
    assert int(cap) == g["capacity"]


@pytest.mark.parametrize("name", ["trio_rr", "trio_fcfs", "trio_oracle", "single_fcfs",
                                  "r0_pascal"])
def test_tiny_goldens_hold_the_reference_test_facts(name):
    """The committed tiny goldens carry the reference tests' literal facts
    (proj/tests/test_engine.cpp:81-179)."""
    lines = open(os.path.join(os.path.dirname(__file__), "golden", name + ".records")).read()
    recs = {}
    for ln in lines.splitlines():
        f = ln.split()
        vals = [float.fromhex(x) for x in f[2:9]]
        nmig = int(f[9])
        k = 10 + 2 * nmig
        nd = int(f[k])
        deliv = [float.fromhex(x) for x in f[k + 1:k + 1 + nd]]
        recs[int(f[1])] = (vals, deliv)
    if name == "trio_rr":
        want = {0: [1, 2, 3, 4, 6, 7, 8, 9], 1: [2, 3, 4, 5, 9, 10, 11, 12],
                2: [5, 6, 7, 8, 10, 11, 12, 13]}
        for i, w in want.items():
            assert recs[i][1] == [float(x) for x in w]
    elif name == "trio_fcfs":
        assert recs[2][0][3] - recs[2][0][0] == 7.0  # C waits 7 units for its first token
    elif name == "trio_oracle":
        for i in range(3):
            assert recs[i][0][3] == recs[i][0][0] + 1.0
    elif name == "single_fcfs":
        v = recs[0][0]
        assert v[1] == pytest.approx(1.0 + 128 * 0.00025)
        assert v[6] == pytest.approx(v[1] + 15 * 0.03)
    elif name == "r0_pascal":
        v = recs[0][0]
        assert v[1] == pytest.approx(0.025) and v[3] == pytest.approx(0.025)
