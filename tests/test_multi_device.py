"""Several GPUs of one process through the C ABI (replicas
shard across GPUs with no data-path collective): pascal_partition_replicas
(host-only, checked here on CPU against its documented rule) and
pascal_run_batch_devices / pascal_sweep_devices (GPU)."""
from __future__ import annotations

import filecmp
import os

import pytest

import paper_2602_11530_b200 as pb

FACTOR = {"pascal": 4.0, "rr": 3.0, "fcfs": 1.0, "oracle": 1.0}


def replicas(n=40):
    traces, cfgs = [], []
    pols = ["pascal", "fcfs", "rr", "oracle"]
    for k in range(n):
        t = pb.Trace.preset("chat", 20 + 7 * (k % 9), 12.0, k)
        traces.append(t)
        cfgs.append(pb.run_config(pols[k % 4], instance_count=2, capacity_fraction=0.5))
    return traces, cfgs


def lpt(traces, cfgs, parts):
    """The documented rule (include/pascal_b200.h): longest-first greedy on
    request-iterations x policy factor (+1 for the oracle capacity pass)."""
    cost = []
    for t, c in zip(traces, cfgs):
        pol = c.policy.decode()
        f = FACTOR[pol] + (1.0 if c.gpu_capacity <= 0 and pol != "oracle" else 0.0)
        cost.append((t.request_iterations() + len(t)) * f)
    order = sorted(range(len(cost)), key=lambda k: (-cost[k], k))
    load = [0.0] * parts
    out = [0] * len(cost)
    for k in order:
        p = min(range(parts), key=lambda q: (load[q], q))
        out[k] = p
        load[p] += cost[k]
    return out, cost


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_partition_is_the_documented_lpt(parts):
    traces, cfgs = replicas()
    got = pb.partition_replicas(traces, cfgs, parts)
    want, cost = lpt(traces, cfgs, parts)
    assert got == want
    assert got == pb.partition_replicas(traces, cfgs, parts)  # deterministic
    loads = [sum(c for c, p in zip(cost, got) if p == q) for q in range(parts)]
    assert max(loads) <= sum(cost) / parts + max(cost)  # LPT bound


def test_partition_rejects_bad_arguments():
    traces, cfgs = replicas(4)
    with pytest.raises(pb.PascalError):
        pb.partition_replicas(traces, cfgs, 0)


@pytest.mark.gpu
def test_run_batch_devices_matches_single_batch():
    traces, cfgs = replicas(24)
    profs = [pb.Profile.default() for _ in traces]
    a = pb.run_batch(traces, profs, cfgs)
    b = pb.run_batch_devices(traces, profs, cfgs, [0])
    for x, y in zip(a, b):
        assert bytes(x) == bytes(y)
    with pytest.raises(pb.PascalError):
        pb.run_batch_devices(traces, profs, cfgs, [0, 0])
    with pytest.raises(pb.PascalError):
        pb.run_batch_devices(traces, profs, cfgs, [64])


@pytest.mark.gpu
def test_sweep_devices_matches_sweep(tmp_path):
    t = pb.Trace.preset("chat", 200, 12.0, 3)
    prof = pb.Profile.default()
    base = pb.run_config("pascal", instance_count=2)
    pb.run_sweep(t, prof, base, ["fcfs", "pascal"], [0.3, 0.6], str(tmp_path / "a"))
    pb.run_sweep(t, prof, base, ["fcfs", "pascal"], [0.3, 0.6], str(tmp_path / "b"), devices=[0])
    names = sorted(os.listdir(tmp_path / "a"))
    assert names == sorted(os.listdir(tmp_path / "b")) and "sweep.csv" in names
    for f in names:
        assert filecmp.cmp(tmp_path / "a" / f, tmp_path / "b" / f, shallow=False), f
