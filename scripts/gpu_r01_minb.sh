# two-row template: __launch_bounds__ min CTAs per SM (SF_JIT_MINB) A/B, configs[4] fp64 + fp32
mkdir -p gpurun_out
SF_JIT_MINB=4 timeout 600 python -m pytest tests/test_gpu_executor.py -q > gpurun_out/minb_tests.log 2>&1; echo "minb4 tests rc=$? $(tail -1 gpurun_out/minb_tests.log)"
for dt in f64 f32; do for r in 2 3; do for m in 1 3 4 5; do
  SF_JIT_MINB=$m timeout 300 python bench.py --workload stencil --radius $r --dtype $dt --steps 5 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err
  python -c "
import json
l=[x for x in open('gpurun_out/c5.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$dt r=$r t=32,16,64 minb=$m', (d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz')) if d else open('gpurun_out/c5.err').read()[-300:])
"
done; done; done 2>&1 | tee gpurun_out/minb_sweep.txt
