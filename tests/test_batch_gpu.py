"""Batched replicas (pascal_batch_*): many different cases in ONE device launch
(mixed trace sizes, instance counts, policies; several replicas per CTA) must
give exactly the per-replica summaries of the reference. The summary.txt a
reference pascal_run would write is rebuilt from each pascal_summary and its
sha256 compared with the golden one."""
import hashlib

import pytest

import paper_2602_11530_b200 as pb
from cases import CASES
from harness import build_trace, golden, make_cfg, make_profile

GOLD = golden()
SMALL = [c for c in CASES if c["name"] in GOLD and c["size"] in ("tiny", "small", "medium")]


def summary_text(c, s):
    cfg = c["cfg"]
    lines = ["pascal-report-v1",
             f"policy={cfg['policy']}",
             f"instance_count={cfg.get('instance_count', 8)}",
             f"gpu_capacity={s.capacity}",
             f"token_quantum={cfg.get('token_quantum', 500)}",
             f"demotion_threshold={cfg.get('demotion_threshold', 5000)}",
             f"no_migration={1 if cfg.get('no_migration') else 0}",
             f"non_adaptive={1 if cfg.get('non_adaptive') else 0}",
             f"requests={s.requests}"]
    for key, v in (("ttft_mean", s.ttft_mean), ("ttft_p50", s.ttft_p50), ("ttft_p90", s.ttft_p90),
                   ("ttft_p95", s.ttft_p95), ("ttft_p99", s.ttft_p99),
                   ("slo_violation_rate", s.slo_violation_rate),
                   ("ttfat_attainment", s.ttfat_attainment), ("throughput", s.throughput)):
        lines.append(f"{key}={v:.9f}")
    return ("\n".join(lines) + "\n").encode()


@pytest.mark.gpu
@pytest.mark.parametrize("repeat", [1, 3])
def test_batch_summaries_match_reference(repeat):
    cases = SMALL * repeat  # repeat > 1: several CTAs run identical replicas concurrently
    traces = [build_trace(c["trace"]) for c in cases]
    profs = [make_profile(c) for c in cases]
    cfgs = [make_cfg(c) for c in cases]
    b = pb.Batch(traces, profs, cfgs)
    for _ in range(2):  # re-execution resets every replica
        b.execute()
        summ = b.summaries()
        bad = []
        for c, s in zip(cases, summ):
            assert s.status == 0, c["name"]
            got = hashlib.sha256(summary_text(c, s)).hexdigest()
            if got != GOLD[c["name"]]["report"]["summary.txt"][0]:
                bad.append(c["name"])
        assert not bad, bad


@pytest.mark.gpu
def test_run_batch_end_to_end_and_histograms():
    cases = [c for c in SMALL if c["name"].startswith("c5_")]
    traces = [build_trace(c["trace"]) for c in cases]
    profs = [make_profile(c) for c in cases]
    cfgs = [make_cfg(c) for c in cases]
    summ = pb.run_batch(traces, profs, cfgs)
    for c, s in zip(cases, summ):
        assert hashlib.sha256(summary_text(c, s)).hexdigest() == \
            GOLD[c["name"]]["report"]["summary.txt"][0]
    b = pb.Batch(traces, profs, cfgs)
    b.set_groups([k % 3 for k in range(len(cases))], 3)
    b.execute()
    hist, slo = b.histograms()
    summ = b.summaries()
    assert sum(map(sum, hist)) == sum(s.requests for s in summ)
    assert sum(v for v, _ in slo) == sum(s.slo_violations for s in summ)
    t = pb.last_timing()
    assert t.engine_ms > 0 and t.kernel_launches >= 4


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{"PB_SMEM": "0"}, {"PB_SMEM": "0", "PB_SMEM_HEAP": "3"},
                                 {"PB_SMEM": "1"}])
def test_launch_shapes_are_bit_exact(env, monkeypatch):
    """Request state in HBM (throughput shape), a 3-slot shared heap that
    must spill to HBM, and full shared-memory residency all give the
    reference's summaries."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cases = [c for c in SMALL if c["size"] != "tiny"]
    traces = [build_trace(c["trace"]) for c in cases]
    b = pb.Batch(traces, [make_profile(c) for c in cases], [make_cfg(c) for c in cases])
    b.execute()
    bad = [c["name"] for c, s in zip(cases, b.summaries())
           if s.status != 0 or hashlib.sha256(summary_text(c, s)).hexdigest() !=
           GOLD[c["name"]]["report"]["summary.txt"][0]]
    assert not bad, bad
