"""Summarise an ncu --set full report into markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep "title" > profiles/xx.md

Per kernel: the headline metrics, DRAM traffic, warp-stall top reasons, and
the hottest source lines (needs -lineinfo builds and --import-source on).
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
           "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
           "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
           "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Occupancy",
           "Achieved Occupancy", "Block Limit Shared Mem", "Block Limit Registers"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "smsp__thread_inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def short(name):
    return name.split("(")[0].split("::")[-1]


def main(rep, title):
    out = io.StringIO()
    out.write(f"# {title}\n\nReport: `{rep}`\n\n")
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index(h) for h in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    det = defaultdict(dict)
    for r in rows[1:]:
        if r[mi] in METRICS:
            det[short(r[ki])][r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    rh = raw[0]
    rawv = defaultdict(dict)
    stalls = defaultdict(list)
    for r in raw[2:]:
        k = short(r[rh.index("Kernel Name")])
        for m in RAW:
            if m in rh:
                rawv[k][m] = r[rh.index(m)]
        for i, h in enumerate(rh):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[k].append((float(r[i].replace(",", "") or 0), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
    for k, v in det.items():
        out.write(f"## {k}\n\n| metric | value |\n|---|---|\n")
        for m in METRICS:
            if m in v:
                out.write(f"| {m} | {v[m]} |\n")
        for m in RAW:
            if m in rawv.get(k, {}):
                out.write(f"| {m} | {rawv[k][m]} |\n")
        st = sorted(stalls.get(k, []), reverse=True)[:6]
        tot = sum(x for x, _ in stalls.get(k, [])) or 1
        if st:
            out.write("\nTop warp-stall reasons (share of samples): " +
                      ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in st) + "\n")
        # Hot source lines.
        src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "-k",
                                              f"regex:{k.split('<')[0]}", "--print-source",
                                              "cuda,sass"))))
        lines, cur, hh = [], None, None
        for r in src:
            if not r:
                continue
            if r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r[0] == "Line No":
                hh = r
                continue
            if hh is None or r[0] == "Function Name" or len(r) < 8 or r[2] != "-":
                continue
            try:
                lines.append((float(r[7] or 0), float(r[4] or 0), f"{cur}:{r[0]}", r[1].strip()[:90]))
            except ValueError:
                pass
        ti = sum(x[0] for x in lines) or 1
        ts = sum(x[1] for x in lines) or 1
        if lines:
            out.write("\n| % inst | % stall | line | source |\n|---|---|---|---|\n")
            for ex, stl, where, text in sorted(lines, reverse=True)[:15]:
                out.write(f"| {100 * ex / ti:.1f} | {100 * stl / ts:.1f} | {where} | `{text}` |\n")
        out.write("\n")
    sys.stdout.write(out.getvalue())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ncu summary")
