#!/bin/bash
# One parameterised GPU session (run under gpurun from the repo root):
#   tools/gpu.sh [tests] [smoke] [bench] [ref] [launches] [ncu] [ab] ...
# tests    pytest -m gpu                       -> gpurun_out/pytest_gpu.log
# smoke    __graft_entry__.smoke()             -> gpurun_out/smoke.log
# bench    python bench.py (default C3 line)   -> gpurun_out/bench.log
# ref      python bench.py --impl reference    -> gpurun_out/bench_ref.log
# launches ncu launch list (time + DRAM bytes) -> gpurun_out/launches.csv
# ncu      ncu --set full of the top kernel    -> gpurun_out/prof_top.ncu-rep
# ab       smoke + tests + short bench for every _lib/exp/*.so variant
# PYTEST_ARGS / BENCH_ARGS / NCU_KERNEL override the defaults.
mkdir -p gpurun_out
NCU_CMD="python bench.py --steps 3 --warmup 3 --preroll 2 --no-cpu --no-e2e ${BENCH_ARGS}"
for what in "$@"; do
  case $what in
    tests) timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
           echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
           echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log ;;
    bench) timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
           tail -1 gpurun_out/bench.log | python tools/line.py ;;
    ref)   timeout 900 python bench.py --impl reference ${BENCH_ARGS} > gpurun_out/bench_ref.log 2>&1
           echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-400 ;;
    launches) timeout 300 $NCU_CMD > gpurun_out/plain.log 2>&1 && \
           timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
             --clock-control none --csv --log-file gpurun_out/launches.csv $NCU_CMD > gpurun_out/ncu_launch.log 2>&1
           echo "launches rc=$?" ;;
    ncu)   timeout 300 $NCU_CMD > gpurun_out/plain2.log 2>&1 && \
           timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_KERNEL:-k_tmem}" \
             -s 6 -c 1 -o gpurun_out/prof_top -f $NCU_CMD > gpurun_out/ncu_full.log 2>&1
           echo "ncu rc=$?" ;;
    ab)    for so in paper_1302_2073_b200/_lib/exp/*.so; do
             echo "== $so"
             export PROST_LIB=$PWD/$so
             timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
             [ -n "$AB_TESTS" ] && timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} 2>&1 | tail -1
             timeout 600 python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 ${BENCH_ARGS} \
               > gpurun_out/ab_$(basename $so).log 2>&1
             tail -1 gpurun_out/ab_$(basename $so).log | python tools/line.py
           done
           unset PROST_LIB ;;
    *) echo "unknown step $what" ;;
  esac
done
