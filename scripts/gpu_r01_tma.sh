mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests2.log 2>&1; echo "tests rc=$?"
timeout 300 python bench.py --no-e2e --no-cpu-baseline --variant tma > gpurun_out/bench_tma.log 2>&1; echo "tma rc=$?"
timeout 300 python bench.py --no-e2e --no-cpu-baseline --variant ldg > gpurun_out/bench_ldg.log 2>&1; echo "ldg rc=$?"
timeout 300 python bench.py --no-e2e --no-cpu-baseline --variant unfused --steps 2 > gpurun_out/bench_unfused.log 2>&1; echo "unfused rc=$?"
