"""Summarize ncu outputs into a markdown file under profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_iter.ncu-rep --rep ... --out profiles/r01_c3_streamed.md --title "..."
"""
import argparse, collections, csv, io, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def launches(path):
    """{kernel: [duration us per launch]} plus {kernel: [dram bytes per launch]}."""
    agg = collections.OrderedDict()
    dram = collections.defaultdict(list)
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        metric = d.get("Metric Name")
        unit = d.get("Metric Unit", "")
        v = float(d["Metric Value"].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            v = v / 1000.0 if unit.startswith("n") else (v if unit.startswith("u") else v * 1000.0)
            agg.setdefault(name, []).append(v)
        elif metric in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            dram[(name, d["ID"])].append(v * scale)
    per = collections.defaultdict(list)
    for (name, _), vs in dram.items():
        per[name].append(sum(vs))
    launches.dram = per
    return agg


def rep(path):
    """Key metrics of a full capture: an .ncu-rep, or its raw-page CSV export
    (tools/ncu_src.sh writes gpurun_out/ncu_raw.csv on the box)."""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                d[label] = f"{vals[i]} {units[i]}".strip()
        kn = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append((kn, d))
    return res


def sass_mix(path, top=14):
    """Executed-instruction mix by opcode and stall reasons (whole kernel)."""
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) >= len(hdr)]

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0
    ops = collections.Counter()
    stalls = collections.Counter()
    scols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for r in data:
        op = r[idx["Source"]].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        ops[o.split(".")[0]] += num(r[idx["Instructions Executed"]])
        for h in scols:
            stalls[h[6:]] += num(r[idx[h]])
    ti, ts = sum(ops.values()) or 1, sum(stalls.values()) or 1
    out = ["## SASS mix and stall reasons (whole kernel)", "",
           f"warp instructions executed: {ti:,}", "",
           "| opcode | share of instructions |", "|---|---|"]
    out += [f"| {k} | {v / ti:.3f} |" for k, v in ops.most_common(top)]
    out += ["", "| stall reason | share of samples |", "|---|---|"]
    out += [f"| {k} | {v / ts:.3f} |" for k, v in stalls.most_common(10)]
    tma = [k for k in ops if k.startswith(("UTMA", "UBLK"))]
    out += ["", f"TMA / bulk-copy opcodes present: {', '.join(tma) if tma else 'none'}", ""]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    ap.add_argument("--sass", default=None, help="SASS source-page CSV: opcode mix + stall reasons")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.note:
        lines += [a.note, ""]
    if a.launches:
        agg = launches(a.launches)
        # only this library's kernels: the benchmark's input generation (torch
        # / cuBLAS) runs before the timed region
        agg = collections.OrderedDict((k, v) for k, v in agg.items() if k.split("::")[-1].startswith("k_"))
        tot = sum(sum(v) for v in agg.values()) or 1.0
        lines += ["## Launch list (ncu `gpu__time_duration.sum`, `--clock-control none`; cold-cache, serialised)", "",
                  "| kernel | launches | avg us | total us | share | DRAM MB / launch |",
                  "|---|---|---|---|---|---|"]
        dram = getattr(launches, "dram", {})
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            d = dram.get(k)
            dm = f"{sum(d) / len(d) / 1e6:.1f}" if d else "-"
            lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {sum(v)/tot:.3f} | {dm} |")
        lines.append("")
    for r in a.rep:
        for kn, d in rep(r):
            lines += [f"## `{kn.split('(')[0]}` (`ncu --set full`, {r.split('/')[-1]})", "", "| metric | value |", "|---|---|"]
            lines += [f"| {k} | {v} |" for k, v in d.items()]
            lines.append("")
    if a.sass:
        lines += sass_mix(a.sass)
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
