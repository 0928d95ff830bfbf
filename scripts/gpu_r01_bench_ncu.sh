mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi2.txt
timeout 600 python bench.py > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --sweeps 20"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_div -s 40 -c 1 -o gpurun_out/prof_sweep $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
