"""Aggregate an ncu source page (--print-source cuda,sass --csv) by CUDA
source line: stall samples and executed instructions."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
stall = defaultdict(float)
inst = defaultdict(float)
text = {}
fname = "?"
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 8 or r[2] != "-":
        continue
    try:
        key = (fname, int(r[0]))
    except ValueError:
        continue
    stall[key] += float(r[4] or 0)
    inst[key] += float(r[7] or 0)
    text[key] = r[1].strip()
ts = sum(stall.values()) or 1
ti = sum(inst.values()) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3e}")
for k in sorted(stall, key=lambda k: -stall[k])[:top]:
    print(f"{100*stall[k]/ts:5.1f}% stall {100*inst[k]/ti:5.1f}% inst  {k[0]}:{k[1]}  {text[k][:90]}")
