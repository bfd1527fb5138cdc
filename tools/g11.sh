mkdir -p gpurun_out
for S in 1 11 22; do
timeout 600 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 --streams $S > gpurun_out/bs_$S.log 2>&1
echo "streams $S"; tail -1 gpurun_out/bs_$S.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.4f' % d['ms_per_step']); print(d.get('resident_counters'))"
done
