# two rows per thread in the TMA tile template (SF_JIT_ROWS=2): parity + configs[4] A/B
mkdir -p gpurun_out
SF_JIT_ROWS=1 timeout 900 python -m pytest tests/test_gpu_executor.py -q -m gpu > gpurun_out/rows1_tests.log 2>&1; echo "rows1 tests rc=$? $(tail -1 gpurun_out/rows1_tests.log)"
SF_JIT_ROWS=2 timeout 900 python -m pytest tests/test_gpu_executor.py -q -m gpu > gpurun_out/rows2_tests.log 2>&1; echo "rows2 tests rc=$? $(tail -1 gpurun_out/rows2_tests.log)"
for dt in f64 f32; do for r in 2 3; do for t in 32,8,64 32,16,64 64,4,64 32,4,64; do for rows in 1 2; do
  [ $dt = f32 ] && [ $t != 32,16,64 ] && [ $t != 32,8,64 ] && continue
  SF_JIT_ROWS=$rows timeout 300 python bench.py --workload stencil --radius $r --tile $t --dtype $dt --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err
  python -c "
import json
l=[x for x in open('gpurun_out/c5.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$dt r=$r t=$t rows=$rows', (d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz')) if d else open('gpurun_out/c5.err').read()[-300:])
"
done; done; done; done 2>&1 | tee gpurun_out/rows2_sweep.txt
