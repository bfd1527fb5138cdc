#!/bin/bash
# A/B of an environment knob on the default bench (alternating runs, same box):
#   AB_VAR=PROST_PREFETCH AB_VALS="0 1" AB_REPS=3 bash tools/ab_env.sh
mkdir -p gpurun_out
for rep in $(seq ${AB_REPS:-3}); do
  for v in ${AB_VALS:-0 1}; do
    env ${AB_VAR}=$v timeout 600 python bench.py --no-cpu --no-e2e --block 0 --steps ${AB_STEPS:-60} --warmup 5 \
      ${BENCH_ARGS} > gpurun_out/ab_${v}_${rep}.log 2>&1
    echo "${AB_VAR}=$v rep=$rep: $(tail -1 gpurun_out/ab_${v}_${rep}.log | python tools/line.py | head -1)"
  done
done
