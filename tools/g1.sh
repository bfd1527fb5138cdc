mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for k in tmem streamed resident; do
PROST_KERNEL=$k timeout 600 python bench.py --no-cpu --steps 10 --warmup 3 > gpurun_out/bench_$k.log 2>&1; echo "bench $k rc=$?"
done
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
for k in tmem streamed resident; do tail -1 gpurun_out/bench_$k.log | cut -c1-600; done
