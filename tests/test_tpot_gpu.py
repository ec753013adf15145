"""Per-request TPOT (north_star: "TTFT/TPOT per request"). The reference
defines no TPOT (proj/src/metrics.cpp:24-83 has TTFT, TTFAT, QoE, blocking);
it is derived from its records: the answer tokens after the first are
delivered over [first_answer_delivery, completion], so
TPOT = (completion - first_answer_delivery) / (A - 1) for A > 1.
The device value must equal that expression evaluated on the reference
records (same two IEEE operations); the rows' other fields must equal the
report the reference writes."""
from __future__ import annotations

import os

import pytest

import paper_2602_11530_b200 as pb
from cases import BY_NAME
from harness import build_trace, make_cfg, make_profile, oracle_run


def records(path):
    out = {}
    with open(path) as f:
        for line in f:
            p = line.split()
            out[int(p[1])] = {"arrival": float.fromhex(p[2]), "first": float.fromhex(p[5]),
                              "completion": float.fromhex(p[8])}
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1_pascal", "c1_fcfs", "r0a1_pascal", "mix500_pascal"])
def test_tpot_rows_match_reference_records(name, tmp_path):
    c = BY_NAME[name]
    t = build_trace(c["trace"])
    rec, _ = oracle_run(c, t, str(tmp_path))
    want = records(rec)
    b = pb.Batch([t], [make_profile(c)], [make_cfg(c)])
    b.execute()
    rows = b.rows(0, len(t))
    s = b.summaries()[0]
    tot, cnt = 0.0, 0
    specs = t.specs()
    for k, row in enumerate(rows):
        A = specs[k][4]
        w = want[row.id]
        assert row.ttft == w["first"] - w["arrival"], (name, k)
        exp = (w["completion"] - w["first"]) / (A - 1) if A > 1 else 0.0
        assert row.tpot == exp, (name, k, row.tpot, exp)
        if A > 1:
            tot += exp
            cnt += 1
    assert s.tpot_requests == cnt
    assert s.tpot_mean == pytest.approx(tot / cnt if cnt else 0.0, rel=1e-12)
