mkdir -p gpurun_out
for d in f32 f64; do for r in 2 3; do for t in 32,8,64 64,4,64 32,8,32; do
  timeout 600 python bench.py --workload stencil --radius $r --dtype $d --tile $t --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err
  python -c "
import json
l=[x for x in open('gpurun_out/c5.json') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$d r=$r t=$t', (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac']) if d else open('gpurun_out/c5.err').read()[-300:])
"
done; done; done
