"""Per-source-line stall / instruction attribution for an ncu --set full report.

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTR [top_n]

ncu's CSV source view has no per-line metrics here, so the SASS rows (in function
order) are zipped with nvdisasm --print-line-info of the same cubin.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_rows(rep, kernel_substr):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kernels, cur, hdr = [], None, None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], []]
            kernels.append(cur)
        elif r and r[0] == "Address":
            hdr = r
        elif cur is not None and hdr is not None and len(r) > 5:
            cur[1].append(dict(zip(hdr, r)))
    for name, rs in kernels:
        if kernel_substr in name:
            return name, rs
    raise SystemExit(f"kernel {kernel_substr!r} not in report: {[k[0][:60] for k in kernels]}")


def line_info(cubin, mangled):
    """(file basename, line) of every SASS instruction of `mangled`, outermost scfa_attn.cu
    frame preferred (inlined helpers are attributed to their call site in the kernel)."""
    out = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    text = out.split(".text." + mangled + ":", 1)[1].split(".section", 1)[0]
    lines, cur = [], None
    for ln in text.splitlines():
        if "//##" in ln:
            locs = re.findall(r'File "([^"]+)", line (\d+)', ln)
            kern = [(os.path.basename(f), int(n)) for f, n in locs if f.endswith("scfa_attn.cu")]
            cur = kern[-1] if kern else (os.path.basename(locs[0][0]), int(locs[0][1])) if locs else cur
            continue
        if re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+[@A-Z]", ln):
            lines.append(cur)
    return lines


def main():
    rep, ksub = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    cubin = sys.argv[4] if len(sys.argv) > 4 else "/tmp/cubin/scfa_attn.sm_100a.cubin"
    name, rows = sass_rows(rep, ksub)
    syms = subprocess.run(["cuobjdump", "-symbols", cubin], capture_output=True, text=True).stdout
    mode = re.search(r"<\(int\)(\d), \(int\)(\d+)>", name)
    want = f"scfa_attn_kernelILi{mode.group(1)}ELi{mode.group(2)}E" if mode else None
    mangled = next(s.split()[-1] for s in syms.splitlines() if want and want in s)
    lines = line_info(cubin, mangled)
    src = open(os.path.join(ROOT, "paper_2306_01160_b200/csrc/scfa_attn.cu")).read().splitlines()
    stall = collections.Counter()
    inst = collections.Counter()
    for i, r in enumerate(rows):
        ln = lines[i] if i < len(lines) else None
        stall[ln] += int(r.get("Warp Stall Sampling (All Samples)", 0) or 0)
        inst[ln] += int(r.get("Instructions Executed", 0) or 0)
    ts, ti = sum(stall.values()), sum(inst.values())
    print(f"{name[:70]}  sass rows {len(rows)} / lineinfo {len(lines)}; samples {ts}, warp-instructions {ti}")
    for ln, c in stall.most_common(top):
        text = src[ln[1] - 1].strip()[:70] if ln and ln[0] == "scfa_attn.cu" else ""
        where = f"{ln[0]}:{ln[1]}" if ln else "?"
        print(f"{c:6d} {100 * c / ts:5.1f}%  inst {100 * inst[ln] / ti:5.1f}%  {where}: {text}")


if __name__ == "__main__":
    main()
