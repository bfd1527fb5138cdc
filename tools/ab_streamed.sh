#!/bin/bash
# A/B the library variants in _lib/exp on the streamed C3 path and C4
for so in paper_1302_2073_b200/_lib/exp/*.so; do
  echo "== $so"
  export PROST_LIB=$PWD/$so
  for c in C3 C4; do
  PROST_KERNEL=streamed timeout 600 python bench.py --config $c --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/abs.log 2>&1
  tail -1 gpurun_out/abs.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c ms/step %.3f  frac %.3f' % (d['ms_per_step'], d['roofline']['frac'])); print({k: round(v['ms_per_step'],3) for k,v in d['phases'].items()})"
  done
done
