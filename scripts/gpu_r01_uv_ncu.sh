mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --sweeps 20"
timeout 300 $CMD > gpurun_out/plain_uv.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_uv.csv $CMD > gpurun_out/ncu_launch_uv.log 2>&1; echo "ncu rc=$?"
