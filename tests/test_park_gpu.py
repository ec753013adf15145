"""The lean Pascal engine parks the all-denied class-1 tail of an instance's
candidates and replays its blocked time later (engine.cu PB_PARK). Blocked
time only reaches the per-request report rows (requests.csv: blocking
latency, QoE inputs), so every Pascal golden case is run through pascal_run
on that build — the instance-parallel engine switched off (PB_PDES=0) so
multi-instance cases take the lean engine too — and all three report files
must be byte-identical to the reference's."""
import os

import pytest

import paper_2602_11530_b200 as pb
from cases import CASES
from harness import build_trace, golden, make_cfg, make_profile, sha_file

GOLD = golden()
PASCAL = [c for c in CASES if c["name"] in GOLD and c["cfg"]["policy"] == "pascal"
          and "report" in GOLD[c["name"]]]
FAST = [c for c in PASCAL if c["size"] in ("tiny", "small", "medium", "large")]
SLOW = [c for c in PASCAL if c["size"] == "xlarge"
        or (c["size"] == "thrash" and (os.environ.get("PB_SLOW")
                                       or (GOLD[c["name"]].get("ref_run_s") or 0) <= 60))]


def _reports_match(c, tmp_path, monkeypatch, smem=None):
    monkeypatch.setenv("PB_PDES", "0")
    if smem is not None:
        monkeypatch.setenv("PB_SMEM", smem)
    g = GOLD[c["name"]]
    t = build_trace(c["trace"])
    prefix = str(tmp_path / "rep")
    pb.run(t, make_profile(c), make_cfg(c), prefix)
    for ext, want in g["report"].items():
        assert sha_file(f"{prefix}.{ext}") == want, ext


@pytest.mark.gpu
@pytest.mark.parametrize("c", FAST, ids=[c["name"] for c in FAST])
def test_lean_pascal_reports(c, tmp_path, monkeypatch):
    _reports_match(c, tmp_path, monkeypatch)


@pytest.mark.gpu
@pytest.mark.parametrize("smem", ["0", "1"])
def test_lean_pascal_reports_c2_shapes(smem, tmp_path, monkeypatch):
    """C2 with request state in HBM (the bench's shape) and in shared memory."""
    _reports_match(next(x for x in PASCAL if x["name"] == "c2_pascal"), tmp_path, monkeypatch,
                   smem)


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("c", SLOW, ids=[c["name"] for c in SLOW])
def test_lean_pascal_reports_xlarge(c, tmp_path, monkeypatch):
    _reports_match(c, tmp_path, monkeypatch)


@pytest.mark.gpu
def test_lean_pascal_batch_rows():
    """Many identical C2 Pascal replicas in one batch (request state in HBM,
    several replicas per warp, warps parking and replaying concurrently): every
    replica's per-request rows, blocked time included, are identical (the
    single-replica runs above pin them to the reference)."""
    c = next(x for x in PASCAL if x["name"] == "c2_pascal")
    t = build_trace(c["trace"])
    k = 64
    b = pb.Batch([t] * k, [make_profile(c)] * k, [make_cfg(c)] * k)
    b.execute()
    summ = b.summaries()
    assert all(s.status == 0 for s in summ)
    def key(r):
        return [(x.ttft, x.ttfat, x.qoe, x.blocking_latency, x.tpot, x.slo_violated)
                for x in b.rows(r, len(t))]
    rows0 = key(0)
    assert any(x[3] > 0 for x in rows0)
    for r in range(1, k, 13):
        assert key(r) == rows0
    assert len({(s.ttft_p99, s.slo_violation_rate) for s in summ}) == 1
