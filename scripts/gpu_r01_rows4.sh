# rows per thread 1/2/4 (SF_JIT_ROWS) after the named-row rewrite: parity + configs[4] A/B
mkdir -p gpurun_out
for rows in 2 4 1; do
SF_JIT_ROWS=$rows timeout 900 python -m pytest tests/test_gpu_executor.py -q -m gpu > gpurun_out/rows${rows}_tests.log 2>&1; echo "rows$rows tests rc=$? $(tail -1 gpurun_out/rows${rows}_tests.log)"
done
for dt in f64 f32; do for r in 2 3; do for t in 32,8,64 32,16,64 64,8,64; do for rows in 1 2 4; do
  SF_JIT_ROWS=$rows timeout 300 python bench.py --workload stencil --radius $r --tile $t --dtype $dt --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err
  python -c "
import json
l=[x for x in open('gpurun_out/c5.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$dt r=$r t=$t rows=$rows', (d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'].get('sm_mhz')) if d else open('gpurun_out/c5.err').read()[-300:])
"
done; done; done; done 2>&1 | tee gpurun_out/rows4_sweep.txt
