# two rows per thread: plane-ring look-ahead (SF_JIT_RING_EXTRA) x tile, configs[4] fp64
mkdir -p gpurun_out
SF_JIT_RING_EXTRA=2 timeout 600 python -m pytest tests/test_gpu_executor.py -q > gpurun_out/ring2_tests.log 2>&1; echo "ring2 tests rc=$? $(tail -1 gpurun_out/ring2_tests.log)"
for r in 2 3; do for t in 32,16,64 32,12,64 32,24,64 64,16,64 32,32,64; do for e in 2 3 4; do
  SF_JIT_RING_EXTRA=$e timeout 300 python bench.py --workload stencil --radius $r --tile $t --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err
  python -c "
import json
l=[x for x in open('gpurun_out/c5.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('f64 r=$r t=$t extra=$e', (d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz')) if d else open('gpurun_out/c5.err').read()[-300:])
"
done; done; done 2>&1 | tee gpurun_out/rows2_ring_sweep.txt
