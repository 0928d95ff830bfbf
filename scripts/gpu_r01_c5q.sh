mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_executor.py -q -m gpu -x > gpurun_out/exec_tests.log 2>&1; echo "exec tests rc=$? $(tail -1 gpurun_out/exec_tests.log)"
for r in 2 3; do
  timeout 600 python bench.py --workload stencil --radius $r --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5_r$r.json 2> gpurun_out/c5_r$r.err
  python -c "
import json
l=[x for x in open('gpurun_out/c5_r$r.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('r=$r', (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac']) if d else open('gpurun_out/c5_r$r.err').read()[-800:])
"
done
