mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/gpu_exec.log 2>&1; echo "exec tests rc=$? $(tail -1 gpurun_out/gpu_exec.log)"
CMD="python bench.py --workload stencil --radius 2 --tile 32,8,64 --steps 2 --warmup 1"
timeout 300 $CMD > gpurun_out/c5plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sf_user_kernel -s 2 -c 1 -o gpurun_out/prof_c5 $CMD > gpurun_out/ncu_c5.log 2>&1; echo "ncu rc=$?"
