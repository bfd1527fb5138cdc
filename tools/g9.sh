mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in C4 C1 C2 C0; do
timeout 600 python bench.py --config $c --no-cpu --steps 10 --warmup 3 > gpurun_out/b_$c.log 2>&1; echo "$c rc=$?"
tail -1 gpurun_out/b_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.3f  value %.1f  frac %.3f e2e %.1f' % (d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['value'])); print(d['config'].get('kernel_path'), {k: round(v['ms_per_step'],3) for k,v in d['phases'].items()})" 2>&1 | tail -2
done
