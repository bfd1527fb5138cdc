# Round profile set (run under gpurun from the repo root): the launch list of
# the default bench's per-frame region (this library's kernels only: time +
# DRAM bytes per launch), then one full capture of a steady-state k_tmem
# launch exported as CSV (tools/ncu_src.sh).
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --block 0 ${BENCH_ARGS}"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k_tmem|k_median|k_combine3|k_pack|k_pass0|k_iter|k_geo|k_stats|k_lsfb|k_gradfb|k_cold|k_xlogic" \
  --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launches rc=$?"
[ -n "$FULL" ] && { BENCH_ARGS="--block 0 ${BENCH_ARGS}" bash tools/ncu_src.sh > /dev/null 2>&1; echo "full rc=$?"; }
ls -la gpurun_out
