mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --sweeps 20"
timeout 300 $CMD > gpurun_out/plain_uv.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_vel_tma -s 2 -c 1 -o gpurun_out/prof_uv $CMD > gpurun_out/ncu_full_uv.log 2>&1; echo "ncu rc=$?"
