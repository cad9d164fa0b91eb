"""Per-source-line instruction / stall shares of one kernel in an ncu report.
Usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
by = sys.argv[4] if len(sys.argv) > 4 else "stall"  # or "inst"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur, hdr, res = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        ex, st = float(r[7] or 0), float(r[4] or 0)
    except ValueError:
        continue
    res.append((ex, st, cur, int(r[0]), r[1].strip()[:90]))
tot = sum(x[0] for x in res) or 1
tst = sum(x[1] for x in res) or 1
print(f"total warp instructions {tot:.3g}; columns: inst% stall%")
for ex, st, f, ln, src in sorted(res, key=lambda x: -(x[0] if by == "inst" else x[1]))[:top]:
    print(f"{ex / tot * 100:5.1f}% {st / tst * 100:5.1f}% {f}:{ln} {src}")
