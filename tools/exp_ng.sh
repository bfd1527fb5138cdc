# A/B of kernel-path switches on the default bench (C3): one line each
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 600 python bench.py --no-cpu --no-e2e --steps 20 --warmup 5 > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log | python tools/line.py
done
