#!/bin/bash
# End-of-round profile set (under gpurun, one GPU): C3 launch list + one full
# k_tmem capture (CSV exports), C4 launch list + one full capture of its
# heaviest kernel.  Outputs: gpurun_out/{c3,c4}_{launches,raw,sass}.csv
mkdir -p gpurun_out
bash tools/prof_round.sh > /dev/null 2>&1; echo "c3 launches rc=$?"
mv gpurun_out/launches.csv gpurun_out/c3_launches.csv
BENCH_ARGS="--block 0" bash tools/ncu_src.sh > /dev/null 2>&1; echo "c3 full rc=$?"
mv gpurun_out/ncu_raw.csv gpurun_out/c3_raw.csv; mv gpurun_out/ncu_sass.csv gpurun_out/c3_sass.csv
BENCH_ARGS="--config C4" bash tools/prof_round.sh > /dev/null 2>&1; echo "c4 launches rc=$?"
mv gpurun_out/launches.csv gpurun_out/c4_launches.csv
NCU_KERNEL="k_geo_tma|k_iter_tma|k_pass0_tma" NCU_SKIP=412 NCU_COUNT=4 BENCH_ARGS="--config C4 --block 0" bash tools/ncu_src.sh > /dev/null 2>&1
echo "c4 full rc=$?"
mv gpurun_out/ncu_raw.csv gpurun_out/c4_raw.csv; mv gpurun_out/ncu_sass.csv gpurun_out/c4_sass.csv
rm -f gpurun_out/ncu_src.csv
ls -la gpurun_out
