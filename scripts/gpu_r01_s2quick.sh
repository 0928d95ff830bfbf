mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "temporal or golden or bench128 or hundred" > gpurun_out/t_q.log 2>&1; rc=$?
echo "tests rc=$rc $(tail -1 gpurun_out/t_q.log)"
if [ $rc -ne 0 ]; then grep -E "^E |FAILED" gpurun_out/t_q.log | head; exit 1; fi
for i in 1 2; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
