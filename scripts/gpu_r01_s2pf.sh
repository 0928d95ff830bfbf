mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "temporal or golden or bench128" > gpurun_out/t_tests.log 2>&1; rc=$?
echo "tests rc=$rc $(tail -1 gpurun_out/t_tests.log)"
if [ $rc -ne 0 ]; then tail -60 gpurun_out/t_tests.log; exit 1; fi
for pf in 0; do
  SF_S2_PF=$pf timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vb.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/vb.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('pf $pf', (d['value'], d['ms_per_step'], d['roofline']['kernel'][:9], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']) if d else open('gpurun_out/vb.log').read()[-600:])
"
done
