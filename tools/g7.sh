mkdir -p gpurun_out
timeout 600 python bench.py --config C4 --no-cpu --steps 10 --warmup 3 > gpurun_out/b_C4.log 2>&1; echo "C4 rc=$?"
tail -1 gpurun_out/b_C4.log | cut -c1-600
timeout 600 python bench.py --config C4 --pixel-shard --no-cpu --steps 10 --warmup 3 > gpurun_out/b_C4p.log 2>&1; echo "C4p rc=$?"
tail -3 gpurun_out/b_C4p.log | cut -c1-1500
timeout 600 python bench.py --config C2 --no-cpu --steps 10 --warmup 3 > gpurun_out/b_C2.log 2>&1; echo "C2 rc=$?"
tail -3 gpurun_out/b_C2.log | cut -c1-600
