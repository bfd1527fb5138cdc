#!/bin/bash
# A/B the library variants in paper_1302_2073_b200/_lib/exp/*.so on the bench,
# in resident and streamed mode
mkdir -p gpurun_out
for so in paper_1302_2073_b200/_lib/exp/*.so; do
  for mode in resident streamed; do
    if [ $mode = streamed ]; then export PROST_NO_RESIDENT=1; else unset PROST_NO_RESIDENT; fi
    echo "== $so $mode"
    PROST_LIB=$PWD/$so timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.3f  value %.0f  frac %.3f' % (d['ms_per_step'], d['value'], d['roofline']['frac'])); print(d.get('resident_counters') or {k:round(v['ms_per_step'],3) for k,v in d['phases'].items()})"
  done
done
