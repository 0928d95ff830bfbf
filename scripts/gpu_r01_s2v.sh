mkdir -p gpurun_out
SF_SWEEP2_VARIANT=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "temporal or golden or bench128 or hundred" > gpurun_out/t_tests_v2.log 2>&1; rc=$?
echo "v2 tests rc=$rc $(tail -1 gpurun_out/t_tests_v2.log)"
if [ $rc -ne 0 ]; then grep -E "^E |FAILED" gpurun_out/t_tests_v2.log | head; fi
for v in 0 2 0 2; do
  SF_SWEEP2_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vb.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/vb.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('v=$v', (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['power_w_max']) if d else open('gpurun_out/vb.log').read()[-600:])
"
done
