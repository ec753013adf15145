"""Replica sweeps sharded across GPUs (BASELINE.json configs[4]).

C5 = 4096 seeds x 16 arrival rates x 4 policies of the acceptance mixed-trace
shape (256 requests, 4 instances, capacity_fraction 0.5,
proj/tests/acceptance.cpp:356-380). Replica id r = (seed * 16 + k) * 4 + p with
lambda_k = 2^(k/3) req/s and p in {pascal, pascal+no_migration,
pascal+non_adaptive, fcfs}. Each rank (one process per GPU) simulates a
contiguous block of replica ids — replicas are independent, so there is no
data-path collective — and the results meet once at the end: one all-gather of
the fixed-size per-replica summaries and one all-reduce(sum) of the
per-(rate, policy) TTFT histograms and SLO counters (NCCL over NVLink on the
GPU box; gloo in the CPU tests).

This module is the host-side driver around the C ABI (`api.Batch`); the
simulations themselves run in the sm_100a engine.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

N_RATES = 16
POLICY_VARIANTS = (
    ("pascal", {}),
    ("pascal_nomig", {"no_migration": 1}),
    ("pascal_nonadaptive", {"non_adaptive": 1}),
    ("fcfs", {}),
)
ACC_CHAT = ("uniform:64:512", "hist:256=0.35,512=0.30,768=0.20,1024=0.10,1536=0.04,2048=0.01",
            "uniform:1024:4096")
ACC_HEAVY = ("uniform:64:512", "uniform:2048:4608", "uniform:128:512")
ACC_PROFILE = {"decode_base": 0.0003, "decode_per_request": 0.001}

# Fields of one per-replica summary record (float64) exchanged by all-gather.
SUMMARY_FIELDS = ("replica", "ttft_mean", "ttft_p50", "ttft_p99", "slo_violation_rate",
                  "throughput", "requests", "request_iterations", "status")


def replica_params(r: int) -> Tuple[int, int, int]:
    """replica id -> (seed, rate index k, policy variant index)."""
    seed, rest = divmod(r, N_RATES * len(POLICY_VARIANTS))
    k, p = divmod(rest, len(POLICY_VARIANTS))
    return seed, k, p


def rate_of(k: int) -> float:
    return 2.0 ** (k / 3.0)


def group_of(r: int) -> int:
    """Histogram group = (rate index, policy variant)."""
    _, k, p = replica_params(r)
    return k * len(POLICY_VARIANTS) + p


def n_groups() -> int:
    return N_RATES * len(POLICY_VARIANTS)


def replica_recipe(r: int, n_requests: int = 256):
    """(trace recipe, run-config fields, profile fields) of replica r."""
    seed, k, p = replica_params(r)
    rate = rate_of(k)
    recipe = {"mix": [{"gen": [n_requests, rate, *ACC_CHAT, seed, False]},
                      {"gen": [n_requests, rate, *ACC_HEAVY, seed + 1, False]}, 0.25, seed + 2]}
    name, extra = POLICY_VARIANTS[p]
    cfg = {"policy": "fcfs" if name == "fcfs" else "pascal", "instance_count": 4,
           "capacity_fraction": 0.5}
    cfg.update(extra)
    return recipe, cfg, dict(ACC_PROFILE)


def policy_cost(p: int) -> float:
    """Relative per-request-iteration cost (FCFS plans are cheaper)."""
    return 0.5 if POLICY_VARIANTS[p][0] == "fcfs" else 1.0


def shard(total: int, world: int, rank: int, weights: Sequence[float] | None = None) -> range:
    """Contiguous block of replica ids for `rank`, balanced by `weights`
    (predicted cost per replica); equal-count blocks when weights is None."""
    if weights is None:
        lo = total * rank // world
        hi = total * (rank + 1) // world
        return range(lo, hi)
    assert len(weights) == total
    pref = [0.0]
    for w in weights:
        pref.append(pref[-1] + w)
    tot = pref[-1]

    def cut(q):  # first index whose prefix reaches q * tot / world
        target = tot * q / world
        lo, hi = 0, total
        while lo < hi:
            mid = (lo + hi) // 2
            if pref[mid] < target:
                lo = mid + 1
            else:
                hi = mid
        return lo

    return range(0 if rank == 0 else cut(rank), total if rank == world - 1 else cut(rank + 1))


# ----------------------------------------------------------------- histograms
HIST_LO, HIST_HI, HIST_BINS = 1e-4, 1e5, 128  # log-spaced TTFT bins (seconds)


def hist_edges() -> List[float]:
    step = (math.log10(HIST_HI) - math.log10(HIST_LO)) / HIST_BINS
    return [10 ** (math.log10(HIST_LO) + i * step) for i in range(HIST_BINS + 1)]


def percentile_from_hist(counts: Sequence[int], pct: float) -> float:
    """Nearest-rank percentile read off a [underflow, bins..., overflow]
    histogram; returns the upper edge of the bin holding rank ceil(p*n)."""
    n = sum(counts)
    if n == 0:
        return 0.0
    rank = max(1, min(n, math.ceil(pct * n)))
    edges = hist_edges()
    acc = 0
    for i, c in enumerate(counts):
        acc += c
        if acc >= rank:
            if i == 0:
                return HIST_LO
            if i == len(counts) - 1:
                return math.inf
            return edges[i]
    return math.inf


def reduce_results(summaries, hist, slo, group=None, device=None):
    """All-gather per-replica summaries ([n_local, len(SUMMARY_FIELDS)] float64)
    and all-reduce(sum) the TTFT histograms ([n_groups, HIST_BINS + 2] int64) and
    SLO counters ([n_groups, 2] int64: violations, requests). Works with NCCL
    (CUDA tensors) and gloo (CPU tensors). Returns global tensors."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return summaries, hist, slo
    world = dist.get_world_size()
    # ragged shards: exchange sizes, pad to the max, gather, trim
    n = torch.tensor([summaries.shape[0]], dtype=torch.int64, device=summaries.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    m = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros((m, summaries.shape[1]), dtype=summaries.dtype, device=summaries.device)
    pad[: summaries.shape[0]] = summaries
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    allsum = torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)])
    h = hist.clone()
    s = slo.clone()
    dist.all_reduce(h, group=group)
    dist.all_reduce(s, group=group)
    return allsum, h, s
