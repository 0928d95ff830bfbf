mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/gpu_tests_q.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_q.log)"
for zc in 64 128 256; do
  SF_ZC=$zc timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vb.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/vb.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('zc $zc', (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']) if d else open('gpurun_out/vb.log').read()[-300:])
"
done
