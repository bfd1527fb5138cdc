"""Markdown table of every config's bench line (tools/configs.sh output).

    python tools/configs_table.py gpurun_out > profiles/r02_configs.md
"""
import json
import sys
from pathlib import Path

d = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out")
print("| config | workload | path | frames/s | ms/frame | e2e frames/s | roofline frac | "
      "blocked frames/s | i_init window frames/s | whole run frames/s | CPU reference frames/s (cores) |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
counters = []
for name in ("C0", "C1", "C2", "C3", "C4", "C4px"):
    p = d / f"cfg_{name}.log"
    if not p.exists():
        continue
    try:
        j = json.loads(p.read_text().strip().splitlines()[-1])
    except Exception:
        continue
    cfg = j.get("config") or {}
    e2e = (j.get("e2e") or {}).get("value")
    blk = (j.get("blocked") or {}).get("value")
    pre = (j.get("preroll") or {}).get("value")
    full = (j.get("full_run") or {}).get("value")
    cpu = j.get("cpu_baseline") or {}
    f = lambda v, fmt="{:.0f}": fmt.format(v) if isinstance(v, (int, float)) else "—"
    print(f"| {name} | {cfg.get('workload', '')} | {cfg.get('kernel_path', '')} | {f(j['value'])} | "
          f"{f(j['ms_per_step'], '{:.4f}')} | {f(e2e)} | {f(j['roofline']['frac'], '{:.3f}')} | {f(blk)} | "
          f"{f(pre)} | {f(full)} | {f(cpu.get('value'), '{:.2f}')} ({cpu.get('cores', '—')}) |")
    if j.get("resident_counters"):
        counters.append((name, j["resident_counters"]))
    if j.get("phases") and not j.get("resident_counters"):
        counters.append((name, {k: round(v["ms_per_step"] * 1000, 1) for k, v in j["phases"].items()}))
print()
print("Per-step counters (TMEM kernel: per-CTA means in µs; streamed: µs per phase per frame, CUDA events"
      " around each launch in a separate pass):")
print()
for name, c in counters:
    print(f"- {name}: " + ", ".join(f"{k} {v}" for k, v in c.items()))
