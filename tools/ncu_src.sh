# Full ncu capture of one steady-state k_tmem launch, exported on the box as
# CSV (the .ncu-rep itself exceeds gpurun's 64 MiB copy-back limit):
#   gpurun_out/ncu_sass.csv  per-SASS-instruction samples / executions
#   gpurun_out/ncu_src.csv   per-CUDA-line aggregates
#   gpurun_out/ncu_raw.csv   all metrics (raw page)
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e ${BENCH_ARGS}"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${NCU_KERNEL:-k_tmem} -s ${NCU_SKIP:-104} -c ${NCU_COUNT:-1} \
  -o /tmp/prof -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass.csv 2>/dev/null
ncu -i /tmp/prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_src.csv 2>/dev/null
ncu -i /tmp/prof.ncu-rep --page raw --csv > gpurun_out/ncu_raw.csv 2>/dev/null
ncu -i /tmp/prof.ncu-rep --page details > gpurun_out/ncu_details.txt 2>/dev/null
ls -la gpurun_out/
