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


# ------------------------------------------------------------------ driver
def select_ids(seeds: int, rates: Sequence[int], policies: Sequence[int]) -> List[int]:
    """Replica ids of the (seed < seeds) x rates x policies sub-grid, ascending."""
    rs, ps = set(rates), set(policies)
    out = []
    for seed in range(seeds):
        for k in range(N_RATES):
            if k not in rs:
                continue
            for p in range(len(POLICY_VARIANTS)):
                if p in ps:
                    out.append((seed * N_RATES + k) * len(POLICY_VARIANTS) + p)
    return out


def run_c5(seeds: int = 4096, rates: Sequence[int] = range(N_RATES),
           policies: Sequence[int] = range(len(POLICY_VARIANTS)), chunk: int = 4736,
           device: int = 0, progress=None):
    """The C5 replica sweep (BASELINE.json configs[4]) on this rank's shard:
    one process per GPU (torch.distributed initialised by the caller, NCCL on
    the GPU box), replicas in device batches of `chunk`, then the end-of-sweep
    exchange (all-gather of per-replica summaries, all-reduce of the
    per-(rate, policy) TTFT histograms and SLO counters). Returns
    (global summaries [n, len(SUMMARY_FIELDS)], histograms, slo, device_ms of
    this rank)."""
    import torch
    import torch.distributed as dist

    from . import api

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    ids = select_ids(seeds, rates, policies)
    weights = [policy_cost(replica_params(r)[2]) for r in ids]
    mine = [ids[j] for j in shard(len(ids), world, rank, weights)]
    api.set_device(device)
    rows = []
    hist = torch.zeros((n_groups(), HIST_BINS + 2), dtype=torch.int64)
    slo = torch.zeros((n_groups(), 2), dtype=torch.int64)
    device_ms = 0.0
    for lo in range(0, len(mine), chunk):
        part = mine[lo:lo + chunk]
        traces, profs, cfgs = [], [], []
        shared = {}  # the policy variants of one (seed, rate) share a trace object, so
        for r in part:  # they also share one oracle capacity pre-run on the device
            recipe, cfg, prof = replica_recipe(r)
            seed, k, _ = replica_params(r)
            if (seed, k) not in shared:
                shared[(seed, k)] = _trace(recipe)
            traces.append(shared[(seed, k)])
            cfgs.append(api.run_config(**cfg))
            profs.append(api.Profile.default(**prof))
        b = api.Batch(traces, profs, cfgs)
        b.set_groups([group_of(r) for r in part], n_groups())
        b.execute()
        device_ms += api.last_timing().total_ms
        summ = b.summaries()
        h, s = b.histograms()
        hist += torch.tensor(h, dtype=torch.int64)
        slo += torch.tensor(s, dtype=torch.int64)
        for r, x in zip(part, summ):
            rows.append([float(r), x.ttft_mean, x.ttft_p50, x.ttft_p99, x.slo_violation_rate,
                         x.throughput, float(x.requests), float(x.request_iterations),
                         float(x.status)])
        del b
        if progress:
            progress(lo + len(part), len(mine))
    t = torch.tensor(rows, dtype=torch.float64).reshape(-1, len(SUMMARY_FIELDS))
    if world > 1:
        dev = torch.device("cuda", device)
        allrows, h, s = reduce_results(t.to(dev), hist.to(dev), slo.to(dev))
        return allrows.cpu(), h.cpu(), s.cpu(), device_ms
    return t, hist, slo, device_ms


def _trace(recipe):
    from . import api

    if "gen" in recipe:
        n, rate, pd, rd, ad, seed, pre = recipe["gen"]
        return api.Trace.generate(n, rate, pd, rd, ad, seed, pre)
    base, repl, frac, seed = recipe["mix"]
    return api.Trace.mix(_trace(base), _trace(repl), frac, seed)


def group_table(hist, slo) -> List[dict]:
    """Per-(rate, policy) rows: TTFT P50/P99 read off the device histogram,
    SLO-violation rate from the counters."""
    out = []
    for g in range(n_groups()):
        k, p = divmod(g, len(POLICY_VARIANTS))
        counts = [int(x) for x in hist[g]]
        n = int(slo[g][1])
        if n == 0:
            continue
        out.append({"rate": rate_of(k), "policy": POLICY_VARIANTS[p][0],
                    "requests": n, "slo_violation_rate": int(slo[g][0]) / n,
                    "ttft_p50_hist": percentile_from_hist(counts, 0.5),
                    "ttft_p99_hist": percentile_from_hist(counts, 0.99)})
    return out


def main(argv=None) -> int:
    """python -m paper_2602_11530_b200.sweep [--seeds S] [--rates K..] [--out CSV]
    (under torchrun for several GPUs: one rank per GPU)."""
    import argparse
    import os

    import torch.distributed as dist

    ap = argparse.ArgumentParser(description="C5 replica sweep (seeds x rates x policies)")
    ap.add_argument("--seeds", type=int, default=64)
    ap.add_argument("--rates", type=int, nargs="+", default=list(range(3, N_RATES)),
                    help="rate indices k (lambda = 2^(k/3)); k < 3 are thrash regimes")
    ap.add_argument("--policies", type=int, nargs="+", default=list(range(len(POLICY_VARIANTS))))
    ap.add_argument("--chunk", type=int, default=4736)
    ap.add_argument("--out", default="c5_sweep.csv")
    a = ap.parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    rows, hist, slo, ms = run_c5(a.seeds, a.rates, a.policies, a.chunk, local)
    if not dist.is_initialized() or dist.get_rank() == 0:
        with open(a.out, "w") as f:
            f.write("rate,policy,requests,slo_violation_rate,ttft_p50_hist,ttft_p99_hist\n")
            for r in group_table(hist, slo):
                f.write(f"{r['rate']:.6f},{r['policy']},{r['requests']},"
                        f"{r['slo_violation_rate']:.6f},{r['ttft_p50_hist']:.6g},"
                        f"{r['ttft_p99_hist']:.6g}\n")
        bad = int((rows[:, 8] != 0).sum()) if rows.numel() else 0
        print(f"{rows.shape[0]} replicas, {int(rows[:, 7].sum()) if rows.numel() else 0} "
              f"request-iterations, device {ms / 1e3:.2f} s on rank 0, failures {bad}; "
              f"wrote {a.out}")
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
