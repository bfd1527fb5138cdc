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
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    if a.note:
        lines += [a.note, ""]
    if a.launches:
        agg = launches(a.launches)
        # only this library's kernels: the benchmark's input generation (torch
        # / cuBLAS) runs before the timed region
        agg = collections.OrderedDict((k, v) for k, v in agg.items() if k.startswith("prost::"))
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
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
