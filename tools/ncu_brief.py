"""Markdown summary of one kernel in an ncu --set full report (raw page).

    python tools/ncu_brief.py REP.ncu-rep --title "..." --algo-bytes N [--out profiles/x.md]
        [--traffic-key NAME --config CONFIG]   # also record DRAM bytes in profiles/ncu_traffic.json
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--title", required=True)
    ap.add_argument("--algo-bytes", type=float, default=0)
    ap.add_argument("--out")
    ap.add_argument("--traffic-key")
    ap.add_argument("--config", default="npb_c")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    name = get.get("Kernel Name", ("?", ""))[0]
    lines = [f"# {a.title}", "", f"Kernel: `{name[:160]}`", ""]
    dur_us = None
    dram = 0.0
    for m in METRICS:
        if m not in get:
            continue
        v, u = get[m]
        lines.append(f"| `{m}` | {v} {u} |") if lines[-1].startswith("|") else lines.extend(["| metric | value |", "|---|---|", f"| `{m}` | {v} {u} |"])
        try:
            f = float(v.replace(",", ""))
        except ValueError:
            continue
        if m == "gpu__time_duration.sum":
            dur_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0) * f
        if m.startswith("dram__bytes"):
            dram += f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    stalls = []
    for h in hdr:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(get[h][0]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    lines += ["", "Warp stalls per issue-active cycle: " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]) + "."]
    if a.algo_bytes and dur_us:
        lines += ["", f"DRAM traffic {dram / 1e6:.1f} MB vs algorithmic {a.algo_bytes / 1e6:.1f} MB per launch "
                      f"({dram / a.algo_bytes:.3f}x); {a.algo_bytes / (dur_us * 1e-6) / 1e9:.0f} GB/s algorithmic "
                      f"over the ncu duration ({dur_us:.1f} us, cold caches, serialised)."]
    if a.note:
        lines += ["", a.note]
    text = "\n".join(lines) + "\n"
    if a.out:
        open(a.out, "w").write(text)
    print(text)
    if a.traffic_key:
        p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {"kernels": {}}
        d["kernels"][a.traffic_key] = {"dram_bytes": dram, "duration_us": dur_us, "round": 2, "config": a.config,
                                       "source": os.path.basename(a.out or "")}
        json.dump(d, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
