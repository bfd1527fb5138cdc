# bench both arms, launch list + one full ncu capture of the frame kernel, cluster probe
mkdir -p gpurun_out
./tools/probe/cluster_probe > gpurun_out/cluster_probe.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --preroll 2 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tmem -s 6 -c 1 -o gpurun_out/prof_tmem -f $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
cat gpurun_out/cluster_probe.log
tail -1 gpurun_out/bench_default.log | cut -c1-300; tail -1 gpurun_out/bench_reference.log | cut -c1-600
