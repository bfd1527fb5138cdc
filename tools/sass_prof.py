"""Summarise an ncu SASS source-page CSV: instructions executed and stall
samples by opcode, and the hottest address ranges.

    ncu -i rep --page source --csv --print-source sass > s.csv; python tools/sass_prof.py s.csv
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex = hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)))
    except (ValueError, IndexError):
        pass
tot_ex = sum(d[2] for d in data)
tot_st = sum(d[3] for d in data)
byop = defaultdict(lambda: [0, 0])
for _, s, ex, st in data:
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    op = op.split(".")[0]
    byop[op][0] += ex
    byop[op][1] += st
print(f"total warp-instr {tot_ex:,}  stall samples {tot_st:,}")
for op, (ex, st) in sorted(byop.items(), key=lambda t: -t[1][0])[:25]:
    print(f"{op:10s} {ex/tot_ex*100:6.2f}% instr  {st/max(tot_st,1)*100:6.2f}% stalls")
# hottest windows of 64 instructions
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
wins = []
for i in range(0, len(data), W):
    seg = data[i:i + W]
    wins.append((sum(d[2] for d in seg), sum(d[3] for d in seg), i))
print("hot windows (start idx, instr%, stall%):")
for ex, st, i in sorted(wins, key=lambda t: -t[0])[:15]:
    print(f"  {i:6d} {ex/tot_ex*100:6.2f}% {st/max(tot_st,1)*100:6.2f}%  first: {data[i][1][:60]}")
