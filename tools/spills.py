"""Local-memory (spill) instructions of one flex kernel instantiation by
source line: python tools/spills.py [KERNEL_SUBSTR] [extra nvcc flags...]"""
import collections
import re
import subprocess
import sys

kern = sys.argv[1] if len(sys.argv) > 1 else "flex_chain_kernelILb0ELi6ELi12E"
src = "paper_1901_06363_b200/csrc/" + ("rigid.cu" if "rigid" in kern else "flex.cu")
extra = sys.argv[2:]
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false",
                "-lineinfo", "-cubin", "-Iinclude", "-Ipaper_1901_06363_b200/csrc", *extra,
                src, "-o", "/tmp/spills.cubin"], check=True)
sass = subprocess.run(["nvdisasm", "--print-line-info", "/tmp/spills.cubin"], capture_output=True,
                      text=True).stdout.splitlines()
on, cur, res, tot = False, None, collections.Counter(), 0
for l in sass:
    if l.startswith(".text."):
        on = kern in l
        continue
    if not on:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        im = re.search(r'inlined at "([^"]+)", line (\d+)', m.group(3))
        if im:
            cur += f" <- {im.group(1).split('/')[-1]}:{im.group(2)}"
        continue
    if re.search(r"\b(LDL|STL)", l):
        res[cur] += 1
        tot += 1
print(f"{tot} local-memory instructions")
for k, v in sorted(res.items(), key=lambda x: -x[1]):
    print(f"{v:4d} {k}")
