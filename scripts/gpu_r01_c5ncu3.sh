mkdir -p gpurun_out
CMD="python bench.py --workload stencil --radius 3 --tile 32,8,64 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/c5plain3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sf_user_kernel -s 3 -c 1 -o gpurun_out/prof_c5r3 $CMD > gpurun_out/ncu_c5r3.log 2>&1; echo "ncu rc=$?"
tail -1 gpurun_out/c5plain3.log | cut -c1-200
