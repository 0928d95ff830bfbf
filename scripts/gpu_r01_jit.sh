mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/gpu_exec.log 2>&1; echo "exec tests rc=$? $(tail -1 gpurun_out/gpu_exec.log)"
SF_JIT_NO_TMA=1 timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/gpu_exec_ldg.log 2>&1; echo "exec tests (no tma) rc=$? $(tail -1 gpurun_out/gpu_exec_ldg.log)"
bash scripts/gpu_r01_c5.sh
