"""Summarise a round's ncu outputs into profiles/ (tracked).

    python tools/ncu_summary.py --round 1 [--launches gpurun_out/launches.csv]
                                [--rep gpurun_out/prof_top.ncu-rep] [--algo-bytes N]

Writes profiles/rNN_launches.md (per-kernel launch count, device time, share of
the profiled window), profiles/rNN_top_kernel.md (key --set full metrics and
stall reasons of the dominant kernel) and profiles/ncu_traffic.json (DRAM bytes
per launch, read by bench.py for roofline.traffic).
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def short(name):
    name = name.replace("b200::<unnamed>::", "").replace("b200::", "")
    return re.sub(r"\(.*", "", name).replace("void ", "")


def launches(path, out, rnd, command="python bench.py --steps 3 --warmup 3 --spmv-reps 10 --no-cpu-baseline "
                                            "--no-verify --no-e2e"):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] == "us":
            v *= 1e3
        elif r["Metric Unit"] == "ms":
            v *= 1e6
        k = short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += v
    total = sum(v[1] for v in agg.values())
    lines = [f"# Round {rnd}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)",
             "", f"Command: `ncu --metrics gpu__time_duration.sum --clock-control none {command}`."
             " Cold-cache, serialised per-launch times: compare shares, not absolutes.",
             "", f"Launches captured: {sum(v[0] for v in agg.values())}, total device time {total/1e6:.3f} ms", "",
             "| kernel | launches | total ms | mean us | share |", "|---|---:|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t/1e6:.3f} | {t/n/1e3:.1f} | {100*t/total:.1f}% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    return agg


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}, vals[hdr.index("Kernel Name")]


def top_kernel(rep, out, rnd, algo_bytes):
    m, kname = raw_metrics(rep)

    def g(k):
        return m.get(k, ("", ""))

    def f(k):
        try:
            return float(g(k)[0].replace(",", ""))
        except ValueError:
            return None

    dur_us = f("gpu__time_duration.sum")
    unit = g("gpu__time_duration.sum")[1]
    if unit == "ns":
        dur_us /= 1e3
    elif unit == "ms":
        dur_us *= 1e3
    rd = f("dram__bytes_read.sum")
    wr = f("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(g("dram__bytes_read.sum")[1], 1)
    wr *= scale.get(g("dram__bytes_write.sum")[1], 1)
    keys = ["dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
    stalls = sorted(((k, f(k)) for k in m if k.startswith("smsp__average_warps_issue_stalled_")
                     and k.endswith("_per_issue_active.ratio") and f(k)), key=lambda kv: -kv[1])[:8]
    lines = [f"# Round {rnd}: top kernel, ncu --set full", "",
             f"Kernel: `{short(kname)}` (`{kname[:160]}`)", "",
             f"* duration: {dur_us:.1f} us (ncu replay, clock-control none)",
             f"* DRAM read {rd/1e6:.1f} MB + write {wr/1e6:.1f} MB = {(rd+wr)/1e6:.1f} MB per launch"
             + (f" vs algorithmic {algo_bytes/1e6:.1f} MB ({(rd+wr)/algo_bytes:.3f}x)" if algo_bytes else ""),
             f"* DRAM bandwidth during the launch: {(rd+wr)/dur_us/1e3:.0f} GB/s", ""]
    lines += ["| metric | value |", "|---|---|"]
    for k in keys:
        v, u = g(k)
        if v:
            lines.append(f"| `{k}` | {v} {u} |")
    lines += ["", "Warp stall reasons (avg warps per issue-active cycle):", "", "| stall | ratio |", "|---|---:|"]
    for k, v in stalls:
        lines.append(f"| {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                     f" | {v:.2f} |")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    d = {}
    if os.path.exists(traffic_path):
        d = json.load(open(traffic_path))
    d.setdefault("kernels", {})[short(kname)] = {"dram_bytes": rd + wr, "duration_us": dur_us,
                                                 "round": rnd, "source": os.path.basename(out)}
    json.dump(d, open(traffic_path, "w"), indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--rep", default=os.path.join(ROOT, "gpurun_out", "prof_top.ncu-rep"))
    ap.add_argument("--algo-bytes", type=float, default=437052704)
    ap.add_argument("--tag", default="")
    ap.add_argument("--command", default=None, help="the profiled command, for the launch list's header")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    tag = f"r{a.round:02d}{a.tag}"
    if os.path.exists(a.launches):
        if a.command:
            launches(a.launches, os.path.join(PROF, f"{tag}_launches.md"), a.round, a.command)
        else:
            launches(a.launches, os.path.join(PROF, f"{tag}_launches.md"), a.round)
    if os.path.exists(a.rep):
        top_kernel(a.rep, os.path.join(PROF, f"{tag}_top_kernel.md"), a.round, a.algo_bytes)


if __name__ == "__main__":
    main()
