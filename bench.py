"""bench.py — scheduled request-iterations/s of the B200 PASCAL scheduling loop.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c2|c1|c5] [--replicas R]

Workload (default c2 = BASELINE.json configs[1]): "4 instances, 2k requests,
Pascal with phase-boundary migration under tight KV-cache budget" — the
reference CLI chat preset (proj/tools/pascalsim_cli.cpp:44-47), 2,000 requests
at lambda = 12 req/s, 4 instances, capacity_fraction 0.3, policy pascal, the
default DS-R1-32B LatencyProfile. One step simulates R independent replicas of
that configuration per GPU (trace seeds 1.., weak scaling), each run to
completion exactly as engine::run does (oracle capacity pre-run + policy run +
metrics); units = request-iterations, identical for every
policy. Multi-GPU: one process per GPU, disjoint seed shards, and one NCCL
all-gather of the per-replica summaries (TTFT percentiles, SLO counters) at the
end of each step; timing is the max over ranks of the device step time.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/ref_dump = /root/reference/proj compiled unmodified; falls back to
the oracle port) on the same workload with all host cores. That arm never
imports this repo's package: its traces come from the reference generator
(`ref_dump gen` / `mix`), and its replicas are a seed prefix of the GPU arm's
(seeds 1..S), run as one longest-first pool of >= 4 replicas per core.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def _load_sweep():
    """paper_2602_11530_b200/sweep.py as a standalone module: replica recipes
    are pure Python, and the reference arm must not import the package (nor
    load libpascal.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_bench_sweep", os.path.join(ROOT, "paper_2602_11530_b200", "sweep.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


sweep = _load_sweep()

METRIC = "scheduled request-iterations/sec (1/2/4/8 B200) + P99 TTFT/SLO match vs CPU ref"
UNIT = "request-iterations/s"
CHAT = ("uniform:64:512", "hist:256=0.35,512=0.30,768=0.20,1024=0.10,1536=0.04,2048=0.01",
        "uniform:256:1024")
ACC_CHAT = ("uniform:64:512", "hist:256=0.35,512=0.30,768=0.20,1024=0.10,1536=0.04,2048=0.01",
            "uniform:1024:4096")
ACC_HEAVY = ("uniform:64:512", "uniform:2048:4608", "uniform:128:512")

# C5 bench slice: rates k >= 3 (lambda >= 2 req/s, the range SURVEY.md §6.3
# measured). At lambda < 2 and capacity 0.5 Pascal replicas enter an
# evict/swap-in thrash regime (the reference ran > 39 CPU-minutes on one).
C5_IDS = [r for r in range(4096 * 64) if sweep.replica_params(r)[1] >= 3]

WORKLOADS = {
    # label: (description, default replicas per GPU)
    # C2: eight replicas per resident warp (8 warps/SM x 148 SMs); the
    # work-stealing loop's end-of-step tail is amortised over twice as many
    # replicas as at four per warp (measured +7.6%, profiles/r2_reps.txt)
    "c2": ("C2: chat preset, 2000 req, lambda 12, 4 instances, capacity_fraction 0.3, pascal",
           9472),
    "c1": ("C1: chat preset, 64 req, lambda 12, 1 instance, capacity_fraction 0.5, pascal", 4736),
    "c5": ("C5 slice: acceptance mixed 256 req, 4 instances, cap 0.5, lambda 2^(k/3) k=3..15, "
           "4 policies, seeds 0..", 4736),
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def replica_specs(workload, rank, per_gpu):
    """(trace recipe, cfg fields, profile fields) for this rank's replicas."""
    out = []
    for k in range(per_gpu):
        g = rank * per_gpu + k
        if workload == "c2":
            out.append(({"gen": [2000, 12.0, *CHAT, 1 + g, False]},
                        dict(policy="pascal", instance_count=4, capacity_fraction=0.3), {}))
        elif workload == "c1":
            out.append(({"gen": [64, 12.0, *CHAT, 1 + g, False]},
                        dict(policy="pascal", instance_count=1, capacity_fraction=0.5), {}))
        else:
            out.append(sweep.replica_recipe(C5_IDS[g]))
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        if shutil.which("nvidia-smi"):
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        busy = [x for x in sm if x > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def algorithmic_bytes(s):
    """B = 16 V + 32 T + 16 T_ans + 16 H + 40 E."""
    return (16 * s.candidate_visits + 32 * s.request_iterations + 16 * s.answer_tokens +
            16 * s.health_checks + 40 * s.events)


def ncu_traffic(workload):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    w = d.get(workload) or {}
    return w.get("dram_bytes_per_launch")


def find_cpu_ref():
    ref = os.path.join(ROOT, "oracle", "_ref", "ref_dump")
    if os.path.exists(ref):
        return ref, "reference"
    port = os.path.join(ROOT, "oracle", "_build", "oracle_dump")
    if not os.path.exists(port):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "restatement"],
                       check=True)
    return port, "port"


def ref_trace_hex(exe, recipe, out, tmp):
    """Materialise a trace recipe with the REFERENCE generator (ref_dump gen /
    mix: proj/src/workload.cpp), never through libpascal.so."""
    if "gen" in recipe:
        n, rate, pd, rd, ad, seed, pre = recipe["gen"]
        subprocess.run([exe, "gen", str(n), repr(float(rate)), pd, rd, ad, str(seed),
                        str(int(pre)), out], check=True)
        return
    base, repl, frac, seed = recipe["mix"]
    a, b = out + ".a", out + ".b"
    ref_trace_hex(exe, base, a, tmp)
    ref_trace_hex(exe, repl, b, tmp)
    subprocess.run([exe, "mix", a, b, repr(float(frac)), str(seed), out], check=True)


def hex_request_iterations(path):
    """SURVEY.md §8d closed form over a pascal-trace-hex-v1 file:
    T = sum(R + A - [R = 0 and not preloaded] + [not preloaded])."""
    t = 0
    with open(path) as f:
        next(f)
        for line in f:
            _, _, _, r, a, pre = line.split()
            r, a, pre = int(r), int(a), int(pre)
            t += r + a - (1 if (r == 0 and not pre) else 0) + (0 if pre else 1)
    return t


def cfg_text(cfg, prof):
    import math
    lines = [f"{k}={v}" for k, v in cfg.items()]
    for k, v in prof.items():
        lines.append(f"{k}={'inf' if math.isinf(float(v)) else repr(float(v))}")
    return "\n".join(lines) + "\n"


def cpu_time_replicas(specs, procs, tmp, outputs=None):
    """Run the CPU reference (`ref_dump sim` = engine::run incl. its capacity
    pre-run) on `specs` with `procs` concurrent processes, handed out
    longest-first from one pool (no step waits on a straggler while cores
    idle); returns (wall seconds, request-iterations). With `outputs` (a
    list), each replica's (ttft_p99, slo_violation_rate, ttft_mean) from the
    reference is appended in spec order."""
    from concurrent.futures import ThreadPoolExecutor

    exe, kind = find_cpu_ref()
    jobs, units, cost = [], 0, []
    for i, (recipe, cfg, prof) in enumerate(specs):
        hexp = os.path.join(tmp, f"r{i}.hex")
        if kind == "reference":
            ref_trace_hex(exe, recipe, hexp, tmp)
        else:  # the C port has no generator: fall back to the product's (checker-side only)
            from harness import build_trace
            build_trace(recipe).save_hex(hexp)
        u = hex_request_iterations(hexp)
        units += u
        cost.append(u * (1 if cfg.get("policy") == "fcfs" else 2))
        cfgp = os.path.join(tmp, f"r{i}.cfg")
        with open(cfgp, "w") as f:
            f.write(cfg_text(cfg, prof))
        jobs.append([exe, "sim", hexp, cfgp])
    order = sorted(range(len(jobs)), key=lambda i: -cost[i])
    res = [None] * len(jobs)

    def one(i):
        r = subprocess.run(jobs[i], capture_output=True, text=True, check=True)
        res[i] = r.stdout

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max(1, procs)) as ex:
        list(ex.map(one, order))
    dt = time.perf_counter() - t0
    if outputs is not None:
        for out in res:
            f = out.split()
            outputs.append(tuple(float.fromhex(x) for x in f[1:4]))
    return dt, units


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU scheduler on all host cores.
    Rank 0 alone runs (the CPU arm does not shard over GPUs); other ranks exit."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    exe, kind = find_cpu_ref()
    desc, _ = WORKLOADS[args.workload]
    # Bounded sample: a seed prefix (1..S) of the GPU arm's replicas, S = 4
    # replicas per host core (>= one per step), run as ONE longest-first pool
    # over all K steps so no step ends waiting on a straggler; the per-step
    # figure is the pool's wall time / K. (One C2 replica is ~10 s on a core,
    # so the whole arm takes ~40 s on 16 cores whatever K is.)
    total = args.ref_replicas or max(4 * cores, args.steps)
    specs = replica_specs(args.workload, 0, total)
    with tempfile.TemporaryDirectory() as tmp:
        for _ in range(args.warmup):  # warm-up: a single small replica (page-in, caches)
            cpu_time_replicas(replica_specs("c1", 0, 1), 1, tmp)
        wall, units = cpu_time_replicas(specs, cores, tmp)
    value = units / wall
    seeds = "seeds 1..%d" % total if args.workload != "c5" else "C5 replica ids %d..%d" % (
        C5_IDS[0], C5_IDS[total - 1])
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference trace generator ref_dump gen/mix, same recipes as the "
                "B200 arm)",
        "config": {"workload": desc, "replicas_total": total, "sample": seeds,
                   "request_iterations_total": units,
                   "timed": "engine::run incl. capacity pre-run, one process per replica, "
                            f"{cores} concurrent, longest-first"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, total),
                         "kind": kind,
                         "sample": f"{total} whole {args.workload} replicas ({seeds}, a prefix "
                                   f"of the B200 arm's), one longest-first pool on {cores} host "
                                   f"cores; ms_per_step = pool wall / steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--replicas", type=int, default=0, help="replicas per GPU per step")
    ap.add_argument("--ref-replicas", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2602_11530_b200 as pb
    from harness import build_trace

    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    pb.set_device(local)
    desc, default_r = WORKLOADS[args.workload]
    per_gpu = args.replicas or default_r
    specs = replica_specs(args.workload, rank, per_gpu)
    traces = [build_trace(r) for r, _, _ in specs]
    cfgs = [pb.run_config(**c) for _, c, _ in specs]
    profs = [pb.Profile.default(**p) for _, _, p in specs]
    units = sum(t.request_iterations() for t in traces)

    # ---- device-resident batch: value (inputs already in HBM)
    batch = pb.Batch(traces, profs, cfgs)
    dev = torch.device("cuda", local)

    base_id = rank * per_gpu
    groups = [sweep.group_of(base_id + k) if args.workload == "c5" else 0
              for k in range(per_gpu)]
    ngroups = sweep.n_groups() if args.workload == "c5" else 1
    batch.set_groups(groups, ngroups)

    def gather(summ):
        """End-of-step exchange: NCCL all-gather of per-replica summaries and
        all-reduce of the device TTFT histograms / SLO counters."""
        h, sl = batch.histograms()
        return gather_from(summ, h, sl)

    def gather_from(summ, h, sl):
        rows = torch.tensor([[float(base_id + k), s.ttft_mean, s.ttft_p50, s.ttft_p99,
                              s.slo_violation_rate, s.throughput, float(s.requests),
                              float(s.request_iterations), float(s.status)]
                             for k, s in enumerate(summ)], dtype=torch.float64)
        h = torch.tensor(h, dtype=torch.int64)
        sl = torch.tensor(sl, dtype=torch.int64)
        if world > 1:
            rows, h, sl = rows.to(dev), h.to(dev), sl.to(dev)
        return sweep.reduce_results(rows, h, sl)

    for _ in range(args.warmup):
        batch.execute()
        gather(batch.summaries())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # A step = simulate (oracle pre-run + policy run + metrics, on the engine's
    # stream; execute() returns when it is done) + the end-of-step exchange
    # (NCCL all-gather / all-reduce on torch's stream at N > 1). The step is
    # bracketed by CUDA events on torch's stream, recorded before the launch
    # and after the collective, so the collective is inside the timed region.
    step_ms, engine_ms, launches = [], [], 0
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            ev0.record()
            batch.execute()
            tm = pb.last_timing()
            summ = batch.summaries()
            grows, ghist, gslo = gather(summ)
            ev1.record()
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            engine_ms.append(tm.engine_ms)
            launches += tm.kernel_launches
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    bad = [s.status for s in summ if s.status != 0]
    if bad:
        raise SystemExit(f"replica failures: {bad[:5]}")
    my_ms = sum(step_ms) / len(step_ms)
    t = torch.tensor([my_ms, sum(engine_ms) / len(engine_ms)], dtype=torch.float64)
    tot_units = units
    if world > 1:
        tt = t.to(dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = tt.cpu()
        u = torch.tensor([units], dtype=torch.float64, device=dev)
        dist.all_reduce(u)
        tot_units = int(u.item())
    ms_step, ms_engine = float(t[0]), float(t[1])
    value = tot_units / (ms_step / 1000.0)
    del batch

    # ---- e2e through the public API with host buffers: trace upload (H2D),
    # simulation, summaries + histograms back (D2H) and, at N > 1, the NCCL
    # exchange, every step
    e2e_times = []
    h2d = d2h = 0
    for i in range(max(1, min(args.steps, 3))):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        b2 = pb.Batch(traces, profs, cfgs)
        tm_up = pb.last_timing()
        b2.set_groups(groups, ngroups)
        b2.execute()
        summ2 = b2.summaries()
        tm2 = pb.last_timing()
        h2, s2 = b2.histograms()
        ex_rows, _, _ = gather_from(summ2, h2, s2)
        if world > 1:
            torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
        h2d = int(tm_up.h2d_bytes)
        d2h = int(tm2.d2h_bytes) + 8 * ngroups * (len(h2[0]) + 2)
        del b2
    e2e_s = torch.tensor([statistics.median(e2e_times)], dtype=torch.float64)
    if world > 1:
        e2e_d = e2e_s.to(dev)
        dist.all_reduce(e2e_d, op=dist.ReduceOp.MAX)
        e2e_s = e2e_d.cpu()
    e2e_value = tot_units / float(e2e_s[0])
    assert [s.ttft_p99 for s in summ2] == [s.ttft_p99 for s in summ]

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline for the dominant kernel (policy-run sched_kernel launch)
    peak, peak_src = load_peaks()
    alg = sum(algorithmic_bytes(s) for s in summ)
    achieved = alg / (ms_engine / 1000.0) / 1e9
    traffic = ncu_traffic(args.workload)
    p99 = sorted(grows[:, 3].tolist())
    tot_slo = gslo.sum(0).tolist()
    slo = tot_slo[0] / max(1, tot_slo[1])
    hist_all = ghist.sum(0).tolist()

    cpu = None
    parity = None
    if not args.no_cpu_baseline and world == 1:
        exe, kind = find_cpu_ref()
        outs = []
        with tempfile.TemporaryDirectory() as tmp:
            dt, u = cpu_time_replicas(specs[:1], 1, tmp, outs)
        cpu = {"value": u / dt, "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"1 whole {args.workload} replica (seed 1), engine::run incl. capacity "
                         f"pre-run, single thread"}
        p99_ref, slo_ref, mean_ref = outs[0]
        s0 = summ[0]
        parity = {"replica": 0, "ttft_p99_gpu": s0.ttft_p99, "ttft_p99_cpu_ref": p99_ref,
                  "slo_violation_rate_gpu": s0.slo_violation_rate,
                  "slo_violation_rate_cpu_ref": slo_ref, "ttft_mean_gpu": s0.ttft_mean,
                  "ttft_mean_cpu_ref": mean_ref,
                  "bit_exact": (s0.ttft_p99, s0.slo_violation_rate, s0.ttft_mean) ==
                               (p99_ref, slo_ref, mean_ref)}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference trace generator, seeds 1..)",
        "config": {"workload": desc, "replicas_per_gpu": per_gpu,
                   "request_iterations_per_step": tot_units,
                   "timed": "oracle capacity pre-run + policy run + metrics on device + "
                            "end-of-step summary/histogram exchange (NCCL at N > 1), CUDA "
                            "events on torch's stream around the whole step",
                   "l2": "inputs larger than L2 (per-replica arenas > 126 MB total)",
                   "parallelism": f"replica shards x{world}"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "timed": "pb.Batch(host traces) upload + execute + summaries/histograms "
                         "download" + (" + NCCL exchange" if world > 1 else "")},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "pb::sched_kernel (policy run)", "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg,
                     "kernel_ms": ms_engine},
        "cpu_baseline": cpu,
        "parity_vs_cpu_ref": parity,
        "clocks": clk.summary(),
        "results": {"replicas_all_ranks": len(p99),
                    "ttft_p99_median_over_replicas": p99[len(p99) // 2],
                    "ttft_p99_from_device_histogram": sweep.percentile_from_hist(hist_all, 0.99),
                    "slo_violation_rate": slo},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
