"""pascalsim-compatible command line over the B200 library.

    python -m paper_2602_11530_b200 gen|run|sweep|compare [options]

Mirrors the reference CLI (proj/tools/pascalsim_cli.cpp; it needs the absent
CLI11 header, so it cannot be built here) option for option and output for
output, on top of the same C ABI. Two differences, both additive:
  * `sweep` simulates every (policy, capacity fraction) point of the grid in
    one device batch (pascal_sweep) instead of one run after another; the files
    it writes are byte-identical to the sequential loop's.
  * `--device N` selects the CUDA device (one process per GPU).
"""
from __future__ import annotations

import argparse
import sys
from typing import Dict, List, Optional

from . import api

RUN_DEFAULTS = dict(policy="pascal", instances=8, capacity=0, capacity_fraction=0.0,
                    quantum=500, demotion_threshold=5000, no_migration=False,
                    non_adaptive=False, target_tpot=0.1, ttfat_target=0.25,
                    qoe_threshold=0.95, pacer_slack=0, profile="")

# (flag dest, config-file key, parser) — proj/tools/pascalsim_cli.cpp:113-138
CONFIG_KEYS = [
    ("policy", "policy", str), ("instances", "instance_count", int),
    ("capacity", "gpu_capacity", int), ("capacity_fraction", "capacity_fraction", float),
    ("quantum", "token_quantum", int), ("demotion_threshold", "demotion_threshold", int),
    ("no_migration", "no_migration", lambda v: v == "1"),
    ("non_adaptive", "non_adaptive", lambda v: v == "1"),
    ("target_tpot", "target_tpot", float), ("ttfat_target", "ttfat_target", float),
    ("qoe_threshold", "qoe_threshold", float), ("pacer_slack", "pacer_slack_tokens", int),
    ("profile", "profile", str),
]


def die(what: str) -> None:
    detail = ""
    try:
        detail = api._lib_().pascal_last_error().decode()
    except Exception:  # noqa: BLE001 - best effort detail, like the reference's die()
        pass
    sys.stderr.write(f"pascalsim: {what}" + (f": {detail}" if detail else "") + "\n")
    sys.exit(1)


def load_config_file(path: str) -> Dict[str, str]:
    """key=value lines, '#' comments (proj/tools/pascalsim_cli.cpp:52-72)."""
    kv = {}
    try:
        lines = open(path).read().split("\n")
    except OSError:
        die("cannot open config file: " + path)
    for line in lines:
        line = line.split("#", 1)[0]
        if "=" not in line:
            continue
        k, v = line.split("=", 1)
        k, v = k.strip(" \t\r"), v.strip(" \t\r")
        if k:
            kv[k] = v
    return kv


def add_run_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--trace", required=True)
    p.add_argument("--config", default="")
    p.add_argument("--profile", default=None)
    p.add_argument("--policy", default=None)
    p.add_argument("--instances", type=int, default=None)
    p.add_argument("--capacity", type=int, default=None)
    p.add_argument("--capacity-fraction", type=float, default=None)
    p.add_argument("--quantum", type=int, default=None)
    p.add_argument("--demotion-threshold", type=int, default=None)
    p.add_argument("--no-migration", action="store_const", const=True, default=None)
    p.add_argument("--non-adaptive", action="store_const", const=True, default=None)
    p.add_argument("--target-tpot", type=float, default=None)
    p.add_argument("--ttfat-target", type=float, default=None)
    p.add_argument("--qoe-threshold", type=float, default=None)
    p.add_argument("--pacer-slack", type=int, default=None)
    p.add_argument("--device", type=int, default=0)


def resolve(a: argparse.Namespace) -> Dict:
    """Flag-over-file resolution (proj/tools/pascalsim_cli.cpp:113-138)."""
    o = dict(RUN_DEFAULTS)
    kv = load_config_file(a.config) if a.config else {}
    for dest, key, conv in CONFIG_KEYS:
        flag = getattr(a, dest)
        if flag is not None:
            o[dest] = flag
        elif key in kv:
            o[dest] = conv(kv[key])
    return o


def make_cfg(o: Dict):
    return api.run_config(
        o["policy"], instance_count=o["instances"], gpu_capacity=o["capacity"],
        capacity_fraction=o["capacity_fraction"], token_quantum=o["quantum"],
        demotion_threshold=o["demotion_threshold"], no_migration=int(o["no_migration"]),
        non_adaptive=int(o["non_adaptive"]), target_tpot=o["target_tpot"],
        ttfat_target=o["ttfat_target"], qoe_threshold=o["qoe_threshold"],
        pacer_slack_tokens=o["pacer_slack"])


def open_profile(path: str) -> api.Profile:
    return api.Profile.load(path) if path else api.Profile.default()


def cmd_gen(a) -> int:
    """proj/tools/pascalsim_cli.cpp:169-222"""
    prompt, reasoning, answering = a.prompt_dist, a.reasoning_dist, a.answering_dist
    preloaded = a.kv_preloaded
    if a.preset:
        if a.preset == "mixed":
            t = api.Trace.preset("mixed", a.count, a.rate, a.seed, a.mix_fraction)
            t.save(a.out)
            print(f"wrote {len(t)} requests to {a.out}")
            return 0
        if a.preset not in api.PRESETS:
            die("unknown preset: " + a.preset)
        p, r, ans, pre = api.PRESETS[a.preset]
        prompt, reasoning, answering = prompt or p, reasoning or r, answering or ans
        preloaded = preloaded or pre
    prompt = prompt or "uniform:64:512"
    reasoning = reasoning or "uniform:128:2048"
    answering = answering or "uniform:128:1024"
    t = api.Trace.generate(a.count, a.rate, prompt, reasoning, answering, a.seed, preloaded)
    if a.mix_trace:
        t = api.Trace.mix(t, api.Trace.load(a.mix_trace), a.mix_fraction, a.seed + 1)
    t.save(a.out)
    print(f"wrote {len(t)} requests to {a.out}")
    return 0


def cmd_run(a) -> int:
    o = resolve(a)
    api.set_device(a.device)
    trace = api.Trace.load(a.trace)
    api.run(trace, open_profile(o["profile"]), make_cfg(o), a.out, a.events or None)
    print(f"wrote {a.out}.{{requests.csv,summary.txt,bins.csv}}")
    return 0


def cmd_sweep(a) -> int:
    """proj/tools/pascalsim_cli.cpp:299-342, one device batch."""
    o = resolve(a)
    fractions: List[float] = a.capacity_fractions or [
        o["capacity_fraction"] if o["capacity_fraction"] > 0 else 0.5]
    api.set_device(a.device)
    trace = api.Trace.load(a.trace)
    api.run_sweep(trace, open_profile(o["profile"]), make_cfg(o), a.policies, fractions, a.out_dir)
    for pol in a.policies:
        for f in fractions:
            print(f"done: {a.out_dir}/{pol}_f{f:.2f}")
    return 0


def cmd_compare(a) -> int:
    names = a.names or a.reports
    if len(names) != len(a.reports):
        die("--names count must match --reports")
    api.compare(a.reports, names, a.out)
    sys.stdout.write(open(a.out).read())
    return 0


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(
        prog="pascalsim", description="deterministic simulator for phase-aware LLM serving "
                                      "policies (B200 engine)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen", help="generate a request trace")
    g.add_argument("--out", default="trace.csv")
    g.add_argument("--count", type=int, default=500)
    g.add_argument("--rate", type=float, default=12.0)
    g.add_argument("--seed", type=int, default=0)
    g.add_argument("--preset", default="")
    g.add_argument("--prompt-dist", default="")
    g.add_argument("--reasoning-dist", default="")
    g.add_argument("--answering-dist", default="")
    g.add_argument("--kv-preloaded", action="store_true")
    g.add_argument("--mix-trace", default="")
    g.add_argument("--mix-fraction", type=float, default=0.5)
    r = sub.add_parser("run", help="simulate one policy over a trace")
    add_run_flags(r)
    r.add_argument("--out", default="report")
    r.add_argument("--events", default="")
    s = sub.add_parser("sweep", help="run a grid of policies and capacities")
    add_run_flags(s)
    s.add_argument("--out-dir", default="sweep")
    s.add_argument("--policies", nargs="+", default=["fcfs", "rr", "oracle", "pascal"])
    s.add_argument("--capacity-fractions", nargs="+", type=float, default=[])
    c = sub.add_parser("compare", help="align reports from the same trace")
    c.add_argument("--reports", nargs="+", required=True)
    c.add_argument("--names", nargs="+", default=[])
    c.add_argument("--out", default="compare.txt")
    a = ap.parse_args(argv)
    if a.cmd == "compare" and len(a.reports) < 2:
        ap.error("--reports needs at least 2 report prefixes")
    try:
        return {"gen": cmd_gen, "run": cmd_run, "sweep": cmd_sweep, "compare": cmd_compare}[
            a.cmd](a)
    except api.PascalError as e:
        die(f"{a.cmd} failed ({e})")
    return 1
