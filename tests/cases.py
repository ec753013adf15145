"""Parity cases shared by oracle/make_golden.py (golden producer, runs the real
reference in this container) and the tests (run the CUDA path on the GPU box).

A case = trace recipe + RunConfig + LatencyProfile. Recipes are either
generator calls (proj/src/workload.cpp generate_trace / mix_traces) or explicit
request tables. Sources of each case are cited next to it.
"""
from __future__ import annotations

import math

CHAT = ("uniform:64:512", "hist:256=0.35,512=0.30,768=0.20,1024=0.10,1536=0.04,2048=0.01",
        "uniform:256:1024")
HEAVY = ("uniform:64:512", "uniform:2048:8192", "uniform:128:512")
# acceptance mixed_trace shape (proj/tests/acceptance.cpp:356-366)
ACC_CHAT = ("uniform:64:512", "hist:256=0.35,512=0.30,768=0.20,1024=0.10,1536=0.04,2048=0.01",
            "uniform:1024:4096")
ACC_HEAVY = ("uniform:64:512", "uniform:2048:4608", "uniform:128:512")

INF = float("inf")


def gen(count, rate, dists, seed, preloaded=False):
    return {"gen": [count, rate, dists[0], dists[1], dists[2], seed, bool(preloaded)]}


def mix(base, repl, fraction, seed):
    return {"mix": [base, repl, fraction, seed]}


def rows(*r):
    """Explicit requests: (id, arrival, prompt, reasoning, answering, preloaded)."""
    return {"rows": [list(x) for x in r]}


def acc_mixed(n, rate, s):
    return mix(gen(n, rate, ACC_CHAT, s), gen(n, rate, ACC_HEAVY, s + 1), 0.25, s + 2)


def cli_mixed(n, rate, s):  # pascalsim gen --preset mixed (pascalsim_cli.cpp:174-193)
    return mix(gen(n, rate, CHAT, s), gen(n, rate, HEAVY, s + 1), 0.25, s + 2)


TRIO = rows(*[(i, float(i), 100, 0, 8, True) for i in range(3)])  # test_engine.cpp:21-34
UNIT = {"prefill_base": 0.0, "prefill_per_token": 0.0, "decode_base": 1.0,
        "swap_bandwidth": INF}                                      # test_engine.cpp:36-43
FAST = {"decode_base": 0.005, "prefill_per_token": 0.00005}        # test_engine.cpp:186-188
FLAT = {"prefill_base": 0.0, "prefill_per_token": 0.0, "decode_base": 0.03}  # acceptance.cpp:222-228
ACC = {"decode_base": 0.0003, "decode_per_request": 0.001}          # acceptance.cpp:378-380


def case(name, trace, policy, profile=None, size="small", **cfg):
    c = {"instance_count": 8, "policy": policy}
    c.update(cfg)
    return {"name": name, "trace": trace, "cfg": c, "profile": dict(profile or {}), "size": size}


CASES = []
# golden contended trio (test_engine.cpp:81-133, acceptance.cpp:76-131)
for pol in ("oracle", "fcfs", "rr", "pascal"):
    CASES.append(case(f"trio_{pol}", TRIO, pol, UNIT, size="tiny", instance_count=1,
                      gpu_capacity=220, token_quantum=4))
# single request closed form (test_engine.cpp:135-158) and R=0 (:160-179)
CASES.append(case("single_fcfs", rows((0, 1.0, 128, 10, 5, False)), "fcfs", size="tiny",
                  instance_count=1))
CASES.append(case("r0_pascal", rows((0, 0.0, 100, 0, 3, False)), "pascal", size="tiny",
                  instance_count=1))
CASES.append(case("r0a1_pascal", rows((0, 0.0, 100, 0, 1, False), (1, 0.01, 50, 0, 1, False)),
                  "pascal", size="tiny", instance_count=2))
# determinism + census traces (test_engine.cpp:181-213, acceptance.cpp:622-671)
for pol in ("fcfs", "rr", "oracle", "pascal"):
    CASES.append(case(f"det77_{pol}",
                      gen(200, 20.0, ("uniform:16:256", "uniform:0:600", "uniform:1:200"), 77),
                      pol, FAST, instance_count=4, capacity_fraction=0.5))
    CASES.append(case(f"det404_{pol}",
                      gen(200, 20.0, ("uniform:16:256", "uniform:0:800", "uniform:1:200"), 404),
                      pol, FAST, instance_count=4, capacity_fraction=0.5))
# ablations (test_engine.cpp:215-234)
ABL = gen(60, 30.0, ("constant:64", "uniform:50:400", "uniform:10:50"), 3)
CASES.append(case("abl60_pascal", ABL, "pascal", {"decode_base": 0.005}, instance_count=3,
                  capacity_fraction=0.4))
CASES.append(case("abl60_nomig", ABL, "pascal", {"decode_base": 0.005}, instance_count=3,
                  capacity_fraction=0.4, no_migration=1))
CASES.append(case("abl60_nonadaptive", ABL, "pascal", {"decode_base": 0.005},
                  instance_count=3, capacity_fraction=0.4, non_adaptive=1))
# C1: chat preset, 64 req, lambda 12, seed 1, 1 instance, cap 0.5
for pol in ("pascal", "fcfs", "rr", "oracle"):
    CASES.append(case(f"c1_{pol}", gen(64, 12.0, CHAT, 1), pol, instance_count=1,
                      capacity_fraction=0.5))
# characterisation runs (acceptance.cpp:247-350)
RCHAR = gen(300, 8.0, ("constant:128", "uniform:128:2048", "constant:1"), 101)
ACHAR = gen(300, 8.0, ("constant:128", "constant:0", "uniform:128:2048"), 202, preloaded=True)
for pol in ("oracle", "fcfs", "rr"):
    CASES.append(case(f"rchar_{pol}", RCHAR, pol, FLAT, instance_count=1, capacity_fraction=0.5))
for pol in ("fcfs", "rr", "pascal"):
    CASES.append(case(f"achar_{pol}", ACHAR, pol, FLAT, instance_count=1, capacity_fraction=0.5))
# acceptance mixed 500 x 8 instances (acceptance.cpp:356-398): 5 policy variants
MIX500 = acc_mixed(500, 12.0, 303)
for name, pol, extra in (("fcfs", "fcfs", {}), ("rr", "rr", {}), ("pascal", "pascal", {}),
                         ("nomig", "pascal", {"no_migration": 1}),
                         ("nonadaptive", "pascal", {"non_adaptive": 1})):
    CASES.append(case(f"mix500_{name}", MIX500, pol, ACC, size="medium", instance_count=8,
                      capacity_fraction=0.5, **extra))
# C5 replica shape: 256 req, 4 instances, lambda 2^(k/3), cap 0.5
for s, k in ((0, 3), (7, 6), (123, 15)):
    rate = 2.0 ** (k / 3.0)
    for name, pol, extra in (("pascal", "pascal", {}), ("nomig", "pascal", {"no_migration": 1}),
                             ("nonadaptive", "pascal", {"non_adaptive": 1}),
                             ("fcfs", "fcfs", {})):
        CASES.append(case(f"c5_s{s}_k{k}_{name}", acc_mixed(256, rate, s), pol, ACC,
                          size="medium", instance_count=4, capacity_fraction=0.5, **extra))
# edge / stress features
CASES.append(case("demote_pascal", gen(120, 10.0, CHAT, 9), "pascal", instance_count=2,
                  capacity_fraction=0.6, demotion_threshold=600))
CASES.append(case("slack_pascal", gen(150, 14.0, CHAT, 11), "pascal", instance_count=3,
                  capacity_fraction=0.5, pacer_slack_tokens=3, target_tpot=0.02))
CASES.append(case("fabric_pascal", gen(150, 14.0, CHAT, 12), "pascal",
                  {"fabric_latency": 0.05, "fabric_bandwidth": 2000.0, "decode_per_kv_token": 1e-6},
                  instance_count=4, capacity_fraction=0.5))
CASES.append(case("infswap_pascal", gen(150, 14.0, CHAT, 13), "pascal",
                  {"swap_bandwidth": INF}, instance_count=3, capacity_fraction=0.4))
CASES.append(case("infswap_rr", gen(150, 14.0, CHAT, 13), "rr", {"swap_bandwidth": INF},
                  instance_count=3, capacity_fraction=0.4))
CASES.append(case("preload_pascal", gen(100, 10.0, CHAT, 14, preloaded=True), "pascal",
                  instance_count=2, capacity_fraction=0.5))
CASES.append(case("preload_rr", gen(100, 10.0, CHAT, 14, preloaded=True), "rr",
                  instance_count=2, capacity_fraction=0.5, token_quantum=37))
CASES.append(case("explicit_cap_pascal", gen(150, 20.0, CHAT, 15), "pascal", instance_count=2,
                  gpu_capacity=3000))
CASES.append(case("tinyq_pascal", gen(80, 6.0, CHAT, 16), "pascal", instance_count=2,
                  capacity_fraction=0.5, token_quantum=7))
CASES.append(case("wide40_pascal", cli_mixed(400, 40.0, 17), "pascal", size="medium",
                  instance_count=40, capacity_fraction=0.5))
CASES.append(case("wide40_fcfs", cli_mixed(400, 40.0, 17), "fcfs", size="medium",
                  instance_count=40, capacity_fraction=0.5))
CASES.append(case("empty_pascal", rows(), "pascal", size="tiny", instance_count=2))
CASES.append(case("tight_pascal", gen(300, 12.0, CHAT, 18), "pascal", size="medium",
                  instance_count=2, capacity_fraction=0.3))
CASES.append(case("tight_nonadaptive", gen(300, 12.0, CHAT, 18), "pascal", size="medium",
                  instance_count=2, capacity_fraction=0.3, non_adaptive=1))
# C2 (BASELINE.json configs[1]): chat 2000 req, lambda 12, 4 instances, cap 0.3, Pascal
CASES.append(case("c2_pascal", gen(2000, 12.0, CHAT, 1), "pascal", size="large",
                  instance_count=4, capacity_fraction=0.3))
CASES.append(case("c2_fcfs", gen(2000, 12.0, CHAT, 1), "fcfs", size="large",
                  instance_count=4, capacity_fraction=0.3))



def cfg_text(c) -> str:
    """key=value config for oracle/ref_dump and oracle/oracle_dump."""
    lines = [f"{k}={v}" for k, v in c["cfg"].items()]
    for k, v in c["profile"].items():
        lines.append(f"{k}={'inf' if (isinstance(v, float) and math.isinf(v)) else repr(float(v))}")
    return "\n".join(lines) + "\n"
# "xlarge": records + report files only (decision logs of 25 M+ lines are not
# materialised). C3 = BASELINE.json configs[2] (ablation, 8 instances, 20k
# requests) at lambda 8, capacity 0.9: Pascal, Pascal(NoMigration), FCFS; and a
# C4-shaped run (configs[3]: CLI mixed preset, 64 instances, long reasoning
# tail) scaled to 20k requests so the CPU reference finishes in seconds.
# (NonAdaptive at this point runs > 15 CPU-minutes on the reference: its
# queues grow without bound; it is covered by the medium ablation cases.)
for name, pol, extra in (("pascal", "pascal", {}), ("nomig", "pascal", {"no_migration": 1}),
                         ("fcfs", "fcfs", {})):
    CASES.append(case(f"c3_l8_{name}", gen(20000, 8.0, CHAT, 1), pol, size="xlarge",
                      instance_count=8, capacity_fraction=0.9, **extra))
CASES.append(case("c4s_pascal", cli_mixed(20000, 16.0, 1), "pascal", size="xlarge",
                  instance_count=64, capacity_fraction=0.9))
CASES.append(case("c4s_fcfs", cli_mixed(20000, 16.0, 1), "fcfs", size="xlarge",
                  instance_count=64, capacity_fraction=0.9))

# C3 across the arrival-rate sweep (BASELINE.json configs[2]: lambda in
# {2, 4, 8, 16}) for all four policy variants, plus the
# stress point lambda = 8 at capacity 0.5 where the reference is O(Q^2).
C3_VARIANTS = (("pascal", "pascal", {}), ("nomig", "pascal", {"no_migration": 1}),
               ("nonadaptive", "pascal", {"non_adaptive": 1}), ("fcfs", "fcfs", {}))
_have = {c["name"] for c in CASES}
for lam in (2, 4, 8, 16):
    for name, pol, extra in C3_VARIANTS:
        if f"c3_l{lam}_{name}" in _have:
            continue
        CASES.append(case(f"c3_l{lam}_{name}", gen(20000, float(lam), CHAT, 1), pol,
                          size="xlarge", instance_count=8, capacity_fraction=0.9, **extra))
for name, pol, extra in C3_VARIANTS:
    CASES.append(case(f"c3x_l8_{name}", gen(20000, 8.0, CHAT, 1), pol, size="xlarge",
                      instance_count=8, capacity_fraction=0.5, **extra))
# C4 at its stated size (BASELINE.json configs[3]: CLI mixed preset,
# pascalsim_cli.cpp:174-193, 1M requests, 64 instances, lambda 16, cap 0.9):
# records sha (piped, never stored) + report files.
for name, pol in (("pascal", "pascal"), ("fcfs", "fcfs")):
    CASES.append(case(f"c4_full_{name}", cli_mixed(1000000, 16.0, 1), pol, size="huge",
                      instance_count=64, capacity_fraction=0.9))
# C5 rates k = 0..2 (lambda = 1, 1.26, 1.59 req/s) at capacity 0.5: the
# evict / swap-in thrash regime (BASELINE.json configs[4]).
for s in (0, 1):
    for k in (0, 1, 2):
        rate = 2.0 ** (k / 3.0)
        for name, pol, extra in C3_VARIANTS:
            CASES.append(case(f"c5_s{s}_k{k}_{name}", acc_mixed(256, rate, s), pol, ACC,
                              size="thrash", instance_count=4, capacity_fraction=0.5, **extra))

BY_NAME = {c["name"]: c for c in CASES}
