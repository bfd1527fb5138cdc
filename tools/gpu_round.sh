#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), launch list, ncu of the top kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 1 --preroll 100 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 1200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_iter|k_geo|k_pass0" -s 1300 -c 4 -o gpurun_out/prof_top -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
