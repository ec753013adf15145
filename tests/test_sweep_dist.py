"""Multi-process (world_size 2, gloo, CPU) checks of the replica-sweep sharding
and the end-of-sweep exchange (paper_2602_11530_b200/sweep.py) — the same code
runs over NCCL on the GPU box."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_11530_b200 import sweep


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    weights = [sweep.policy_cost(sweep.replica_params(r)[2]) for r in range(total)]
    mine = sweep.shard(total, world, rank, weights)
    # fake per-replica results, deterministic in the replica id
    rows = torch.tensor([[float(r), r * 0.5, r * 0.25, r * 1.0, (r % 7) / 7.0, 100.0 + r, 256.0,
                          1000.0 + r, 0.0] for r in mine], dtype=torch.float64)
    hist = torch.zeros((sweep.n_groups(), sweep.HIST_BINS + 2), dtype=torch.int64)
    slo = torch.zeros((sweep.n_groups(), 2), dtype=torch.int64)
    for r in mine:
        g = sweep.group_of(r)
        hist[g, 1 + r % sweep.HIST_BINS] += 1
        slo[g, 0] += r % 3
        slo[g, 1] += 256
    allrows, h, s = sweep.reduce_results(rows, hist, slo)
    out_q.put((rank, list(mine), allrows[:, 0].tolist(), h.sum().item(), s.sum(0).tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [64, 1000])
def test_two_rank_exchange(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    shards = [r[1] for r in res]
    assert shards[0] + shards[1] == list(range(total))  # disjoint, contiguous, complete
    for _, _, ids, hsum, ssum in res:
        assert ids == [float(r) for r in range(total)]  # all-gather in rank order
        assert hsum == total
        assert ssum == [sum(r % 3 for r in range(total)), 256 * total]


def test_shard_balances_cost():
    total = 4096
    w = [sweep.policy_cost(sweep.replica_params(r)[2]) for r in range(total)]
    parts = [sweep.shard(total, 8, k, w) for k in range(8)]
    assert sum(len(p) for p in parts) == total
    costs = [sum(w[r] for r in p) for p in parts]
    assert max(costs) - min(costs) <= 1.0


def test_replica_ids_round_trip():
    for r in (0, 1, 63, 64, 4096 * 64 - 1):
        seed, k, p = sweep.replica_params(r)
        assert (seed * 16 + k) * 4 + p == r
    assert sweep.rate_of(0) == 1.0 and sweep.rate_of(15) == 32.0
    hist = [0] * (sweep.HIST_BINS + 2)
    hist[10] = 99
    hist[100] = 1
    assert sweep.percentile_from_hist(hist, 0.5) == sweep.hist_edges()[10]
    assert sweep.percentile_from_hist(hist, 1.0) == sweep.hist_edges()[100]


def test_select_ids_and_group_table():
    ids = sweep.select_ids(3, [3, 15], [0, 3])
    assert len(ids) == 3 * 2 * 2 and ids == sorted(ids)
    assert {sweep.replica_params(r)[1] for r in ids} == {3, 15}
    assert {sweep.replica_params(r)[2] for r in ids} == {0, 3}
    hist = torch.zeros((sweep.n_groups(), sweep.HIST_BINS + 2), dtype=torch.int64)
    slo = torch.zeros((sweep.n_groups(), 2), dtype=torch.int64)
    g = sweep.group_of(ids[0])
    hist[g, 20] = 10
    slo[g] = torch.tensor([3, 10])
    rows = sweep.group_table(hist, slo)
    assert len(rows) == 1 and rows[0]["policy"] == "pascal" and rows[0]["rate"] == 2.0
    assert rows[0]["slo_violation_rate"] == 0.3
    assert rows[0]["ttft_p99_hist"] == sweep.hist_edges()[20]


@pytest.mark.gpu
def test_c5_subgrid_matches_reference(tmp_path):
    """run_c5 on 2 seeds x 2 rates x 4 policies: every replica's P99 TTFT,
    SLO-violation rate and mean TTFT equal the reference's (oracle/_ref)."""
    import subprocess

    from cases import cfg_text
    from harness import REF_DUMP, build_trace

    if not os.path.exists(REF_DUMP):
        pytest.skip("reference not built")
    rows, hist, slo, _ = sweep.run_c5(seeds=2, rates=[4, 12], chunk=5)
    assert rows.shape[0] == 16 and int((rows[:, 8] != 0).sum()) == 0
    assert int(slo[:, 1].sum()) == 16 * 256
    for row in rows.tolist():
        recipe, cfg, prof = sweep.replica_recipe(int(row[0]))
        t = build_trace(recipe)
        hexp, cfgp = str(tmp_path / "t.hex"), str(tmp_path / "c.cfg")
        t.save_hex(hexp)
        with open(cfgp, "w") as f:
            f.write(cfg_text({"cfg": cfg, "profile": prof}))
        out = subprocess.run([REF_DUMP, "sim", hexp, cfgp], check=True, capture_output=True,
                             text=True, timeout=300).stdout.split()
        p99, slo_rate, mean = (float.fromhex(x) for x in out[1:4])
        assert (row[3], row[4], row[1]) == (p99, slo_rate, mean), row
