mkdir -p gpurun_out
for pf in 0 2 1; do
PROST_PREFETCH=$pf timeout 600 python bench.py --no-cpu --no-e2e --steps 20 --warmup 3 > gpurun_out/b5_$pf.log 2>&1
echo "prefetch $pf"; tail -1 gpurun_out/b5_$pf.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.3f  value %.0f  frac %.3f' % (d['ms_per_step'], d['value'], d['roofline']['frac'])); print(d.get('resident_counters'))"
done
