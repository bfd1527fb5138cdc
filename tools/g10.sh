mkdir -p gpurun_out
for w in 0 16 24 32; do
PROST_KERNEL=streamed timeout 600 python bench.py --no-cpu --no-e2e --steps 10 --warmup 3 --wave $w > gpurun_out/bw_$w.log 2>&1
echo "wave $w"; tail -1 gpurun_out/bw_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/step %.3f  frac %.3f' % (d['ms_per_step'], d['roofline']['frac'])); print({k: round(v['ms_per_step'],3) for k,v in d['phases'].items()})"
done
