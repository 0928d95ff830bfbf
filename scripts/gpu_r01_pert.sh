mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "periodic or temporal or golden or bench128" > gpurun_out/pert_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/pert_tests.log)"
grep -E "Error|assert" gpurun_out/pert_tests.log | head -5
for sd in 2026 7; do timeout 500 python scripts/probes/parity_stress.py 1500 $sd 250 > gpurun_out/parity_pert_$sd.log 2>&1; echo "seed $sd rc=$? $(tail -1 gpurun_out/parity_pert_$sd.log)"; grep DIFF gpurun_out/parity_pert_$sd.log | head -5; done
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
