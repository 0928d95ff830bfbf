# default (no minimum CTAs/SM) vs SF_JIT_MINB 1/3/4 on the same box, after making the minimum opt-in
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_executor.py -q > gpurun_out/exec_tests.log 2>&1; echo "exec tests rc=$? $(tail -1 gpurun_out/exec_tests.log)"
for r in 2 3; do for m in unset 1 3 4; do
  if [ $m = unset ]; then E=""; else E="SF_JIT_MINB=$m"; fi
  env $E timeout 300 python bench.py --workload stencil --radius $r --steps 5 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err
  python -c "
import json
l=[x for x in open('gpurun_out/c5.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('f64 r=$r t=32,16,64 minb=$m', (d['roofline']['avg_launch_ms'], d['roofline']['frac']) if d else open('gpurun_out/c5.err').read()[-300:])
"
done; done 2>&1 | tee gpurun_out/minb2_sweep.txt
