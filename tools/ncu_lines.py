"""Aggregate an ncu source export (tools/ncu_src.sh: gpurun_out/ncu_src.csv)
per CUDA source line: share of warp-stall samples and of executed warp
instructions, top N lines.  python tools/ncu_lines.py [csv] [N]"""
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu_src.csv"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


agg, cur, idx = {}, None, None
for r in csv.reader(open(path)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        idx = {h: i for i, h in enumerate(r)}
        continue
    if r[0] == "Function Name" or idx is None or r[0] == "":
        continue
    s = num(r[idx["Warp Stall Sampling (All Samples)"]])
    n = num(r[idx["Instructions Executed"]])
    agg[(cur, num(r[0]))] = (s, n, r[1])
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts}  warp instructions {ti}")
for (f, line), (s, n, src) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{f:22s} {line:5d} samp {s / ts:6.3f} inst {n / ti:6.3f}  {src.strip()[:80]}")
