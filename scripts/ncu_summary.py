"""Summarise an ncu --set full capture of pb::sched_kernel into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep LABEL [--workload c2]

Writes profiles/<LABEL>.md (key metrics, stall mix, hottest source lines) and,
with --workload, records the DRAM bytes of the launch in
profiles/ncu_summary.json (read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], check=True, capture_output=True,
                          text=True).stdout


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * mult.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("label")
    ap.add_argument("--workload")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    rows = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    raw = {h[i]: (v[i], u[i]) for i in range(len(h))}
    src = list(csv.reader(io.StringIO(ncu(a.rep, "--page", "source", "--csv",
                                          "--print-source", "cuda,sass"))))
    hdr = src[2]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_i = hdr.index("Instructions Executed")
    stall_cols = [i for i, x in enumerate(hdr) if x.startswith("stall_") and "Not Issued" not in x]
    lines, stalls = [], {hdr[i]: 0 for i in stall_cols}
    for r in src[3:]:
        if len(r) <= max(i_s, i_i) or not r[0]:
            continue
        try:
            lines.append((int(r[i_s]), int(r[i_i]), int(r[0]), r[1].strip()[:100]))
        except ValueError:
            continue
        for i in stall_cols:
            try:
                stalls[hdr[i]] += int(r[i])
            except ValueError:
                pass
    tot_s = sum(x[0] for x in lines) or 1
    tot_i = sum(x[1] for x in lines) or 1
    st = sum(stalls.values()) or 1
    dram = to_bytes(*raw["dram__bytes_read.sum"]) + to_bytes(*raw["dram__bytes_write.sum"])
    out = [f"# ncu summary: {a.label}", "", a.note, "", f"source: `{os.path.basename(a.rep)}`", "",
           "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        if k in raw:
            out.append(f"| {k} | {raw[k][0]} | {raw[k][1]} |")
    out += ["", f"DRAM bytes (read + write) for the launch: {dram:.4g}", "",
            "## Stall mix (all samples)", "", "| reason | share |", "|---|---|"]
    for k, val in sorted(stalls.items(), key=lambda x: -x[1])[:10]:
        out.append(f"| {k} | {100 * val / st:.1f}% |")
    out += ["", "## Hottest source lines (stall samples / instructions)", "",
            "| samples | instr | line | source |", "|---|---|---|---|"]
    for s, i, ln, text in sorted(lines, reverse=True)[:30]:
        out.append(f"| {100 * s / tot_s:.1f}% | {100 * i / tot_i:.1f}% | {ln} | `{text}` |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", a.label + ".md"), "w") as f:
        f.write("\n".join(out) + "\n")
    if a.workload:
        p = os.path.join(ROOT, "profiles", "ncu_summary.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[a.workload] = {"dram_bytes_per_launch": dram, "profile": a.label,
                         "kernel_s": float(raw["gpu__time_duration.sum"][0])}
        with open(p, "w") as f:
            json.dump(d, f, indent=1)
    print("\n".join(out[:40]))


if __name__ == "__main__":
    main()
