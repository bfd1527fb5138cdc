mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/b3.log 2>&1
tail -1 gpurun_out/b3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.3f  value %.0f  frac %.3f' % (d['ms_per_step'], d['value'], d['roofline']['frac'])); print(d.get('resident_counters'), d['config'].get('kernel_path'))"
