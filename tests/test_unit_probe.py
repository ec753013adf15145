"""Plan-level and placement-level parity (SURVEY.md §8c unit seams).

The reference unit-tests its planner and placement rules as pure functions on
hand-built states (proj/tests/test_instance.cpp:84-306,
proj/tests/test_cluster.cpp:67-107, proj/tests/acceptance.cpp:137-216). The
device engine fuses them into its event loop; `pb.probe_maybe_start` /
`pb.probe_select` run the engine's own planner / select_instance for one step
on such a state (include/pascal_b200.h "Unit-parity seams").

* the reference's planner fixtures, restated with their own expected values;
* a forced free < 0 repair (proj/src/instance.cpp:233-243);
* randomised states: device step vs the REAL reference's apply_demotion +
  plan_iteration + maybe_start application (oracle/_ref/ref_dump plan);
* every snapshot vector of acceptance.cpp criterion 2 (1,087,080) through the
  device select_instance vs the reference's cluster functions
  (oracle/_ref/ref_dump select).
"""
from __future__ import annotations

import math
import os
import random
import subprocess

import numpy as np
import pytest

import paper_2602_11530_b200 as pb
from harness import REF_DUMP

INF = math.inf


def R(**kw):
    return kw


# ---------------------------------------------------------------- fixtures
@pytest.mark.gpu
def test_demotion_strict_and_resets_round_robin_state():
    # test_instance.cpp:84-110: kv 5000 stays, 5001 demoted, quanta reset, seq 11
    reqs = [R(prompt=10, reasoning=9000, answering=1, phase="reasoning", kv=kv, quanta=3,
              qused=17, loc="cpu", tokens=kv - 10) for kv in (5000, 5001, 4999)]
    out = pb.probe_maybe_start(reqs, [0, 1, 2], [], gpu_capacity=0, cpu_used=15000,
                               enqueue_counter=10, demotion_threshold=5000)
    assert out["demoted"] == [1]


@pytest.mark.gpu
def test_planner_prefill_is_a_dedicated_iteration():
    # test_instance.cpp:146-161
    prof = pb.Profile.default(prefill_base=0.0, prefill_per_token=0.001)
    out = pb.probe_maybe_start([R(prompt=100, reasoning=5, answering=5)], [0], [],
                               gpu_capacity=1000, policy="fcfs", profile=prof)
    assert out["kind"] == "prefill" and out["prefill_request"] == 0
    assert out["batch"] == []
    assert out["completion_time"] == pytest.approx(0.1)


@pytest.mark.gpu
def test_planner_decode_batches_residents_and_prices_the_step():
    # test_instance.cpp:163-184
    prof = pb.Profile.default(decode_base=0.03, decode_per_kv_token=1e-5)
    reqs = [R(prompt=100, reasoning=10, answering=10, phase="reasoning", kv=150, tokens=50)
            for _ in range(2)]
    out = pb.probe_maybe_start(reqs, [0, 1], [], gpu_capacity=1000, gpu_used=300,
                               policy="fcfs", profile=prof)
    assert out["kind"] == "decode" and len(out["batch"]) == 2
    assert out["completion_time"] == pytest.approx(0.03 + 1e-5 * 300)
    assert out["evictions"] == [] and out["denied"] == []


@pytest.mark.gpu
def test_planner_fcfs_blocks_strictly_behind_the_head():
    # test_instance.cpp:186-208
    reqs = [R(prompt=200, reasoning=50, answering=5, phase="reasoning", kv=200),
            R(prompt=100, reasoning=5, answering=5),
            R(prompt=10, reasoning=5, answering=5)]
    out = pb.probe_maybe_start(reqs, [0, 1, 2], [], gpu_capacity=250, gpu_used=200,
                               policy="fcfs")
    assert out["kind"] == "decode" and out["batch"] == [0]
    assert out["evictions"] == []
    assert sorted(out["denied"]) == [1, 2]


@pytest.mark.gpu
def test_planner_rr_evicts_the_most_exhausted_resident():
    # test_instance.cpp:210-233
    prof = pb.Profile.default(swap_bandwidth=INF)
    reqs = [R(prompt=100, reasoning=0, answering=8, phase="answering", kv=104, tokens=4,
              quanta=1),
            R(prompt=100, reasoning=0, answering=8, phase="answering", kv=100, loc="cpu")]
    out = pb.probe_maybe_start(reqs, [0, 1], [], gpu_capacity=180, gpu_used=104, cpu_used=100,
                               policy="rr", profile=prof)
    assert out["evictions"] == [0]
    assert out["immediate_swap_ins"] == [1]
    assert out["batch"] == [1]


@pytest.mark.gpu
def test_planner_phase_priority_protects_the_high_class():
    # test_instance.cpp:235-265 (both parts)
    reqs = [R(prompt=100, reasoning=50, answering=5, phase="reasoning", kv=104),
            R(prompt=100, reasoning=0, answering=8, phase="answering", kv=104, seq=1)]
    out = pb.probe_maybe_start(reqs, [0], [1], gpu_capacity=208, gpu_used=208,
                               enqueue_counter=1)
    assert out["batch"] == [0] and out["evictions"] == [1]
    reqs[1]["loc"] = "cpu"
    out = pb.probe_maybe_start(reqs, [0], [1], gpu_capacity=208, gpu_used=104, cpu_used=104,
                               enqueue_counter=1)
    assert out["batch"] == [0] and out["evictions"] == []
    assert 1 in out["denied"]


@pytest.mark.gpu
def test_planner_oracle_admits_everything():
    # test_instance.cpp:267-283 (KV sizes scaled into the engine's 2^26 token range)
    reqs = [R(prompt=100, reasoning=10, answering=10, phase="reasoning", kv=1000000)
            for _ in range(16)]
    out = pb.probe_maybe_start(reqs, list(range(16)), [], gpu_capacity=(2**63 - 1) // 4,
                               gpu_used=16 * 1000000, policy="oracle")
    assert len(out["batch"]) == 16 and out["evictions"] == [] and out["denied"] == []


@pytest.mark.gpu
def test_planner_swapping_and_in_transit_are_not_candidates():
    # test_instance.cpp:285-306
    reqs = [R(prompt=100, reasoning=10, answering=10, phase="reasoning", kv=100,
              swapping_out=True, loc="cpu"),
            R(prompt=100, reasoning=10, answering=10, phase="answering", kv=100, loc="transit",
              seq=1)]
    out = pb.probe_maybe_start(reqs, [0], [1], gpu_capacity=1000, enqueue_counter=1)
    assert out["kind"] == "idle"


@pytest.mark.gpu
def test_planner_over_capacity_repair_fires():
    # instance.cpp:233-243: KV growth left the oracle's residents 5 tokens over;
    # nothing is admitted, so the repair evicts in reverse arrival order
    reqs = [R(prompt=10, reasoning=100, answering=10, phase="reasoning", kv=50),
            R(prompt=10, reasoning=100, answering=10, phase="reasoning", kv=55)]
    out = pb.probe_maybe_start(reqs, [0, 1], [], gpu_capacity=100, gpu_used=105,
                               policy="oracle", profile=pb.Profile.default(swap_bandwidth=INF))
    assert out["evictions"] == [1]
    assert out["gpu_used"] == 50 and not out["over_capacity"]
    assert sorted(out["denied"]) == [0, 1] and out["kind"] == "idle"


# ------------------------------------------------- random states vs reference
PROF_KEYS = ("prefill_base", "prefill_per_token", "decode_base", "decode_per_request",
             "decode_per_kv_token", "swap_bandwidth")


def random_state(rng: random.Random, policy: str):
    n = rng.choice([1, 3, 8, 31, 33, 64, 90])
    reqs = []
    for k in range(n):
        P, Rt, A = rng.randint(1, 400), rng.choice([0, 0, 50, 300, 900]), rng.randint(1, 300)
        phase = rng.choice(["waiting", "reasoning", "answering", "answering"])
        if phase == "reasoning" and Rt == 0:
            phase = "answering"
        r = R(prompt=P, reasoning=Rt, answering=A, phase=phase)
        if phase == "waiting":
            r.update(kv=0, loc="gpu", tokens=0)
        else:
            tok = rng.randint(0, Rt - 1) if phase == "reasoning" else Rt + rng.randint(0, A - 1)
            r["tokens"] = tok
            r["kv"] = P + tok + rng.choice([0, 0, 1])
            loc = rng.choice(["gpu", "gpu", "cpu", "cpu", "transit"])
            r["loc"] = loc
            if loc == "cpu":
                s = rng.random()
                if s < 0.15:
                    r["swapping_in"] = True
                elif s < 0.3:
                    r["swapping_out"] = True
            elif loc == "gpu" and rng.random() < 0.05:
                r["kv"] = 0
        r["quanta"] = rng.choice([0, 0, 1, 2, 3]) if rng.random() < 0.9 else rng.randint(0, 40)
        r["qused"] = rng.randint(0, 20)
        reqs.append(r)
    high, low = [], []
    seq = 0
    # enqueue order: baselines enqueue only at arrival (their queue is in
    # arrival order, engine.cpp:111-116,260-283); Pascal's low queue fills in
    # event order (transitions, demotions, transfers)
    order = rng.sample(range(n), n) if policy == "pascal" else list(range(n))
    for k in order:
        if rng.random() < 0.1:
            continue  # not queued
        r = reqs[k]
        seq += rng.randint(1, 3)
        r["seq"] = seq
        to_low = policy == "pascal" and (r["phase"] == "answering" or rng.random() < 0.2)
        (low if to_low else high).append(k)
    for k in range(n):
        if k not in high and k not in low:
            r = reqs[k]
            r["seq"] = 0
            if rng.random() < 0.5:
                r["phase"] = "done"
    res_kv = sum(r.get("kv", 0) for r in reqs
                 if r["phase"] != "done" and (r.get("loc") == "gpu" or r.get("swapping_in")))
    cpu_kv = sum(r.get("kv", 0) for r in reqs if r["phase"] != "done" and r.get("loc") == "cpu"
                 and not r.get("swapping_in"))
    gpu_used = res_kv + rng.choice([0, 0, 0, 1, 3, 40])
    cap = max(0, gpu_used + rng.choice([-30, -4, 0, 5, 60, 200, 900, 5000]))
    if policy == "oracle" and rng.random() < 0.5:
        cap = 10**12
    prof = {"prefill_base": rng.choice([0.0, 0.01]),
            "prefill_per_token": rng.choice([0.00025, 0.001]),
            "decode_base": rng.choice([0.03, 0.0003]),
            "decode_per_request": rng.choice([0.0, 0.001]),
            "decode_per_kv_token": rng.choice([0.0, 1e-5]),
            "swap_bandwidth": rng.choice([INF, 51200.0, 2000.0])}
    st = dict(requests=reqs, high=high, low=low, gpu_capacity=cap, gpu_used=gpu_used,
              cpu_used=cpu_kv, policy=policy, enqueue_counter=seq + rng.randint(0, 5),
              demotion_threshold=rng.choice([5000, 300, 120]),
              now=rng.choice([0.0, 1.5, 1234.0625]),
              candidate_scratch=rng.choice([0, 16, 256]))
    return st, prof


PHASE_NUM = {"waiting": 0, "reasoning": 1, "answering": 2, "done": 4}
LOC_NUM = {"gpu": 0, "cpu": 1, "transit": 2}


def ref_plan(st, prof, tmp):
    path = os.path.join(tmp, "state.txt")
    with open(path, "w") as f:
        for k in ("policy",):
            f.write(f"{k} {st[k]}\n")
        f.write(f"capacity {st['gpu_capacity']}\ngpu_used {st['gpu_used']}\n"
                f"cpu_used {st['cpu_used']}\ncounter {st['enqueue_counter']}\n"
                f"demotion {st['demotion_threshold']}\nnow {float(st['now']).hex()}\n")
        for k, v in prof.items():
            f.write(f"prof {k} {'inf' if math.isinf(v) else float(v).hex()}\n")
        for k, r in enumerate(st["requests"]):
            f.write("req {} {} {} {} {} {} {} {} {} {} {} {} {}\n".format(
                float(k).hex(), r.get("prompt", 1), r.get("reasoning", 0), r.get("answering", 1),
                PHASE_NUM[r.get("phase", "waiting")], LOC_NUM[r.get("loc", "gpu")],
                int(bool(r.get("swapping_in"))), int(bool(r.get("swapping_out"))),
                r.get("tokens", 0), r.get("kv", 0), r.get("qused", 0), r.get("quanta", 0),
                r.get("seq", 0)))
        f.write("high " + " ".join(map(str, st["high"])) + "\n")
        f.write("low " + " ".join(map(str, st["low"])) + "\n")
    p = subprocess.run([REF_DUMP, "plan", path], capture_output=True, text=True, timeout=30)
    assert p.returncode == 0, p.stderr
    out = {}
    for line in p.stdout.splitlines():
        parts = line.split()
        out[parts[0]] = parts[1:]
    ints = lambda k: [int(x) for x in out[k]]  # noqa: E731
    ev = out["swapev"]
    return {"demoted": ints("demoted"), "evictions": ints("evict"), "swap_ins": ints("swapin"),
            "immediate_swap_ins": ints("immediate"), "denied": ints("denied"),
            "kind": ("idle", "prefill", "decode")[int(out["kind"][0])],
            "prefill_request": int(out["kind"][2]), "batch": ints("batch"),
            "gpu_used": int(out["used"][0]), "cpu_used": int(out["used"][1]),
            "completion_time": float.fromhex(out["completion"][0]),
            "swap_events": [(int(ev[i]), float.fromhex(ev[i + 1])) for i in range(0, len(ev), 2)],
            "blocked": float.fromhex(out["blocked"][0]), "over_capacity": out["over"][0] == "1"}


FIELDS = ("demoted", "evictions", "swap_ins", "immediate_swap_ins", "denied", "kind", "batch",
          "gpu_used", "cpu_used", "completion_time", "swap_events", "over_capacity")


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["pascal", "rr", "fcfs", "oracle"])
def test_random_plan_steps_match_reference(policy, tmp_path):
    if not os.path.exists(REF_DUMP):
        pytest.skip("reference not built (oracle/_ref)")
    rng = random.Random(2602 + ("pascal", "rr", "fcfs", "oracle").index(policy))
    for trial in range(150):
        st, prof = random_state(rng, policy)
        want = ref_plan(st, prof, str(tmp_path))
        got = pb.probe_maybe_start(profile=pb.Profile.default(**prof), **st)
        for k in FIELDS:
            assert got[k] == want[k], (trial, k, got[k], want[k], st, prof)
        if want["kind"] == "prefill":
            assert got["prefill_request"] == want["prefill_request"]
        den = set(want["denied"])
        for k, b in enumerate(got["blocked"]):
            assert b == (want["blocked"] if k in den else 0.0), (trial, k)


def test_ref_plan_tool_on_reference_fixtures(tmp_path):
    """Pins the checker: ref_dump plan reproduces the reference's own fixture
    expectations (test_instance.cpp:186-233) on this CPU."""
    if not os.path.exists(REF_DUMP):
        pytest.skip("reference not built (oracle/_ref)")
    reqs = [R(prompt=200, reasoning=50, answering=5, phase="reasoning", kv=200),
            R(prompt=100, reasoning=5, answering=5),
            R(prompt=10, reasoning=5, answering=5)]
    st = dict(requests=reqs, high=[0, 1, 2], low=[], gpu_capacity=250, gpu_used=200,
              cpu_used=0, policy="fcfs", enqueue_counter=0, demotion_threshold=5000, now=0.0)
    out = ref_plan(st, {}, str(tmp_path))
    assert out["kind"] == "decode" and out["batch"] == [0] and sorted(out["denied"]) == [1, 2]
    reqs = [R(prompt=100, reasoning=0, answering=8, phase="answering", kv=104, tokens=4,
              quanta=1),
            R(prompt=100, reasoning=0, answering=8, phase="answering", kv=100, loc="cpu")]
    st = dict(requests=reqs, high=[0, 1], low=[], gpu_capacity=180, gpu_used=104, cpu_used=100,
              policy="rr", enqueue_counter=0, demotion_threshold=5000, now=0.0)
    out = ref_plan(st, {"swap_bandwidth": INF}, str(tmp_path))
    assert out["evictions"] == [0] and out["immediate_swap_ins"] == [1] and out["batch"] == [1]
    rng = random.Random(7)
    for policy in ("pascal", "rr", "fcfs", "oracle"):  # the generator's states are accepted
        for _ in range(5):
            st, prof = random_state(rng, policy)
            ref_plan(st, prof, str(tmp_path))


# ---------------------------------------------- placement rules, exhaustive
def criterion2_vectors():
    """The snapshot vectors of acceptance.cpp criterion 2 (:168-216), in order."""
    reas, ans = [], []
    for n in range(1, 5):
        codes = np.arange(8 ** n)
        t = np.zeros((len(codes), n), np.uint8)
        m = np.zeros((len(codes), n), np.int64)
        c = codes.copy()
        for i in range(n):
            t[:, i] = c % 2
            c //= 2
            m[:, i] = c % 4
            c //= 4
        reas.append((t, m))
    for n in range(1, 5):
        codes = np.arange(32 ** n)
        t = np.zeros((len(codes), n), np.uint8)
        r = np.zeros((len(codes), n), np.int64)
        a = np.zeros((len(codes), n), np.int64)
        c = codes.copy()
        for i in range(n):
            t[:, i] = c % 2
            c //= 2
            r[:, i] = c % 4
            c //= 4
            a[:, i] = c % 4
            c //= 4
        ans.append((t, r, a))
    return reas, ans


@pytest.mark.gpu
def test_placement_exhaustive_vs_reference(tmp_path):
    if not os.path.exists(REF_DUMP):
        pytest.skip("reference not built (oracle/_ref)")
    path = str(tmp_path / "sel.bin")
    subprocess.run([REF_DUMP, "select", path], check=True, timeout=120)
    want = np.fromfile(path, dtype=np.uint8)
    reas, ans = criterion2_vectors()
    got = []
    for mode in (0, 2):
        for t, m in reas:
            got.append(pb.probe_select(mode, t, m))
    for t, r, a in ans:
        got.append(pb.probe_select(1, t, r, a))
    got = np.concatenate(got).astype(np.uint8)
    assert len(got) == len(want) == 2 * 4680 + 1082400
    bad = np.nonzero(got != want)[0]
    assert len(bad) == 0, f"{len(bad)} vectors differ, first at {bad[:5]}"


@pytest.mark.gpu
def test_placement_ties_and_wide_clusters():
    # test_cluster.cpp:109-118: equal snapshots pick the lowest id; plus a 32-
    # instance vector (one lane per instance) with the healthy minimum last
    t = np.ones((1, 2), np.uint8)
    assert pb.probe_select(0, t, np.array([[5, 5]]))[0] == 0
    assert pb.probe_select(1, t, np.array([[2, 2]]), np.array([[1, 1]]))[0] == 0
    t = np.zeros((1, 32), np.uint8)
    t[0, 31] = 1
    m = np.arange(32, 0, -1)[None, :].astype(np.int64) + 10
    m[0, 31] = 100
    assert pb.probe_select(0, t, m)[0] == 31      # Alg. 1: healthy wins over smaller m
    assert pb.probe_select(2, t, m)[0] == 30      # baseline: plain argmin m
