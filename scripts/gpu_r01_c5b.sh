mkdir -p gpurun_out/jit
timeout 600 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/gpu_exec.log 2>&1; echo "exec tests rc=$? $(tail -1 gpurun_out/gpu_exec.log)"
: > gpurun_out/c5.log
for r in 2 3; do
  for t in 32,8,64 64,4,64 32,16,64 32,4,64; do
    SF_JIT_DUMP=gpurun_out/jit timeout 300 python bench.py --workload stencil --radius $r --tile $t --steps 5 --warmup 2 > gpurun_out/c5b.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/c5b.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('r $r tile $t', (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['achieved'], d['roofline']['frac'], d['clocks']['sm_mhz']) if d else open('gpurun_out/c5b.log').read()[-400:])
" >> gpurun_out/c5.log
  done
done
