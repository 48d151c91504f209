"""Opcode histogram and hottest instructions of an ncu --page source --csv --print-source sass export."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iS, iW, iE = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iE]), int(r[iW]), r[iS].strip()))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
totw = sum(d[1] for d in data) or 1
print("instructions", tot, "stall samples", totw)
c, cw = Counter(), Counter()
for e, w, src in data:
    op = (src.split()[1] if src.startswith("@") else src.split()[0]).split(".")[0]
    c[op] += e
    cw[op] += w
for op, e in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} {e:>11d} {100 * e / tot:5.1f}%  stall {100 * cw[op] / totw:5.1f}%")
print("-- hottest (stall samples)")
for e, w, src in sorted(data, key=lambda d: -d[1])[:15]:
    print(f"{w:6d} {e:>10d}  {src[:80]}")
