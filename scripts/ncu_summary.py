"""Summarise a gpurun profiling session into profiles/ (tracked).

    python scripts/ncu_summary.py --tag r01_baseline [--rep gpurun_out/prof_attn.ncu-rep]
        [--launches gpurun_out/launches.csv] [--bench gpurun_out/bench.json]

Writes profiles/<tag>.md (launch-list shares, per-kernel ncu --set full metrics and
stall reasons) and updates profiles/ncu_traffic.json (DRAM bytes per launch of each
attention entry point, read by bench.py for roofline.traffic).
"""

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODE_NAME = {"0": "scfa_attn_fwd", "1": "scfa_attn_bwd_dq", "2": "scfa_attn_bwd_dkdv", "3": "scfa_attn_bwd"}
METRICS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "MB read"),
    ("dram__bytes_write.sum", "MB write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu (MUFU) %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "cyc/inst"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def kernel_label(name):
    if "scfa_attn_kernel<" in name:
        mode = name.split("scfa_attn_kernel<")[1].split(",")[0].replace("(int)", "").strip()
        d = name.split("scfa_attn_kernel<")[1].split(",")[1].split(">")[0].replace("(int)", "").strip()
        return f"{MODE_NAME.get(mode, mode)} (D={d})"
    return name.split("(")[0].replace("void ", "")


def launches_table(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    per = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi and r[vi]:
            per[kernel_label(r[ki])].append(float(r[vi].replace(",", "")) / 1000.0)
    total = sum(sum(v) for v in per.values())
    out = ["| kernel | launches | avg us | total us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {100 * sum(v) / total:.1f}% |")
    return "\n".join(out)


def ncu_raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--rep", default=os.path.join(ROOT, "gpurun_out", "prof_attn.ncu-rep"))
    ap.add_argument("--launches", default=os.path.join(ROOT, "gpurun_out", "launches.csv"))
    ap.add_argument("--bench", default=os.path.join(ROOT, "gpurun_out", "bench.json"))
    ap.add_argument("--note", default="")
    ap.add_argument("--no-traffic", action="store_true", help="do not update profiles/ncu_traffic.json")
    a = ap.parse_args()
    md = [f"# Profile {a.tag}", ""]
    if a.note:
        md += [a.note, ""]
    if os.path.exists(a.bench):
        line = open(a.bench).read().strip().splitlines()[-1]
        md += ["## bench.py line (not under a profiler)", "", "```json", line, "```", ""]
    if os.path.exists(a.launches):
        md += ["## Launch list (ncu gpu__time_duration, cold-cache, serialised: compare shares)", "",
               launches_table(a.launches), ""]
    traffic = {}
    if os.path.exists(a.rep):
        h, units, rows = ncu_raw(a.rep)
        col = {c: i for i, c in enumerate(h)}
        md += ["## ncu --set full of the attention kernels", "",
               "| kernel | " + " | ".join(u for _, u in METRICS) + " |",
               "|---|" + "---|" * len(METRICS)]
        stall_cols = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
        stall_md = []
        for r in rows:
            name = kernel_label(r[col["Kernel Name"]])
            vals = []
            for m, _ in METRICS:
                v = r[col[m]] if m in col else ""
                try:
                    f = float(v.replace(",", ""))
                    unit = units[col[m]] if m in col else ""
                    if m == "gpu__time_duration.sum":  # to microseconds whatever ncu chose
                        f *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
                              "s": 1e6}.get(unit, 1.0)
                    elif m.startswith("dram__bytes"):  # to MB
                        f *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
                    vals.append(f"{f:.1f}")
                except ValueError:
                    vals.append(v)
            md.append(f"| {name} | " + " | ".join(vals) + " |")
            try:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = float(r[col["dram__bytes_read.sum"]].replace(",", "")) * scale[units[col["dram__bytes_read.sum"]]]
                wr = float(r[col["dram__bytes_write.sum"]].replace(",", "")) * scale[units[col["dram__bytes_write.sum"]]]
                traffic.setdefault(name.split(" ")[0], rd + wr)
            except (KeyError, ValueError):
                pass
            st = sorted(((float(r[col[c]] or 0), c.replace("smsp__pcsamp_warps_issue_stalled_", "")) for c in stall_cols),
                        reverse=True)[:6]
            stall_md.append(f"- {name}: " + ", ".join(f"{n} {int(v)}" for v, n in st))
        md += ["", "Top warp-stall samples per kernel:", ""] + stall_md + [""]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    if traffic and not a.no_traffic:
        path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        old = json.load(open(path)) if os.path.exists(path) else {}
        old.update(traffic)
        old["_source"] = a.tag
        json.dump(old, open(path, "w"), indent=1, sort_keys=True)
    print("\n".join(md))


if __name__ == "__main__":
    main()
