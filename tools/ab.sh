#!/bin/bash
# A/B the library variants in paper_1302_2073_b200/_lib/exp/*.so: smoke + parity
# tests + bench (default kernel path), one line each.
mkdir -p gpurun_out
for so in paper_1302_2073_b200/_lib/exp/*.so; do
  echo "== $so"
  export PROST_LIB=$PWD/$so
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
  timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
  timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 "$@" > gpurun_out/ab_$(basename $so).log 2>&1
  tail -1 gpurun_out/ab_$(basename $so).log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.3f  value %.0f  frac %.3f' % (d['ms_per_step'], d['value'], d['roofline']['frac'])); print(d.get('resident_counters'), d['config'].get('kernel_path'))"
done
