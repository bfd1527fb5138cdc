#!/bin/bash
# Every BASELINE config on one GPU (under gpurun): gpurun_out/cfg_<name>.log,
# then python tools/configs_table.py gpurun_out > profiles/rNN_configs.md
mkdir -p gpurun_out
for c in C0 C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-30} --warmup 5 > gpurun_out/cfg_$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/cfg_$c.log | python tools/line.py | head -1
done
timeout 900 python bench.py --config C4 --pixel-shard --steps 20 --warmup 4 --no-cpu --no-e2e \
  > gpurun_out/cfg_C4px.log 2>&1
echo "C4px rc=$?"; tail -1 gpurun_out/cfg_C4px.log | python tools/line.py | head -1
