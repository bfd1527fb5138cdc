mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --preroll 2 --no-cpu --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu c3 rc=$?"
CMD4="python bench.py --config C4 --steps 3 --warmup 3 --preroll 2 --no-cpu --no-e2e"
timeout 300 $CMD4 > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD4 > gpurun_out/ncu_launch4.log 2>&1; echo "ncu c4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter -s 20 -c 1 -o gpurun_out/prof_c4_iter -f $CMD4 > gpurun_out/ncu_full4.log 2>&1; echo "ncu c4 full rc=$?"
