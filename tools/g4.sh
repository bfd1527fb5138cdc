mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --preroll 2 --no-cpu --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tmem -s 6 -c 1 -o gpurun_out/prof_tmem3 -f $CMD > gpurun_out/ncu_full3.log 2>&1; echo "ncu rc=$?"
