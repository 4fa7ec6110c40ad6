"""Per-source-line instruction and stall totals of one kernel in an ncu report (run here, no GPU).

ncu's SASS source page (absolute addresses) is joined with nvdisasm's line table of the same kernel in the
.so that was profiled (offsets from the kernel entry).

    python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_MANGLED [label:first-last ...]
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
from pathlib import Path

rep, lib, kern = sys.argv[1:4]
ranges = []
for spec in sys.argv[4:]:
    name, span = spec.split(":")
    a, b = span.split("-")
    ranges.append((name, int(a), int(b)))

src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hdr_i]
ix = {x: i for i, x in enumerate(h)}
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
addrs = [int(r[ix["Address"]], 16) for r in data]
base = min(addrs)

# ranges are line spans of march.cu (lines of other files -- headers, inlined library code -- are listed below)
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(lib).resolve())], cwd=td, capture_output=True, check=True)
    off2line = {}
    for cub in Path(td).glob("*.cubin"):
        dis = subprocess.run(["nvdisasm", "-g", "-c", str(cub)], capture_output=True, text=True).stdout
        sec = dis.find(f".text.{kern}:")
        if sec < 0:
            continue
        end = dis.find("//---------------------", sec)
        line = ("?", 0)
        for l in dis[sec:end if end > 0 else None].splitlines():
            m = re.search(r'//## File "(.*)", line (\d+)', l)
            if m:
                line = (Path(m.group(1)).name, int(m.group(2)))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
            if m:
                off2line[int(m.group(1), 16)] = line
        break

inst = collections.Counter()
stall = collections.Counter()
for r, a in zip(data, addrs):
    ln = off2line.get(a - base, ("?", -1))
    inst[ln] += float(r[ix["Instructions Executed"]] or 0)
    stall[ln] += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
T, S = sum(inst.values()), sum(stall.values())
print(f"total warp instructions {T:.4g}, stall samples {S:.0f}, lines mapped {len(inst)}")
if ranges:
    for name, a, b in ranges:
        i = sum(v for k, v in inst.items() if k[0] == "march.cu" and a <= k[1] <= b)
        s = sum(v for k, v in stall.items() if k[0] == "march.cu" and a <= k[1] <= b)
        print(f"{name:24s} lines {a}-{b}: {i / T * 100:5.1f} % instr, {s / S * 100:5.1f} % stall samples")
for ln in sorted(inst, key=lambda k: -inst[k])[:40]:
    print(f"{ln[0]}:{ln[1]:<5d} {inst[ln] / T * 100:5.1f} % instr  {stall[ln] / S * 100:5.1f} % stall")
