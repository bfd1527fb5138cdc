"""Summarise one bench.py JSON line from stdin (used by tools/gpu.sh)."""
import json
import sys

raw = sys.stdin.read().strip()
try:
    d = json.loads(raw)
except Exception:
    print("no JSON line:", raw[-300:])
    sys.exit(0)
r = d.get("roofline") or {}
e = d.get("e2e") or {}
c = d.get("cpu_baseline") or {}
print(f"value {d.get('value', 0):.0f} {d.get('unit')}  ms/step {d.get('ms_per_step', 0):.4f}  "
      f"frac {r.get('frac', 0):.3f}  e2e {e.get('value')}  cpu {c.get('value')}  "
      f"clocks {d.get('clocks')}")
print("path:", (d.get("config") or {}).get("kernel_path"), " counters:", d.get("resident_counters"))
