mkdir -p gpurun_out
: > gpurun_out/stages.log
for v in 0 9 10 11; do
  SF_SWEEP_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ten_steps or projection or odd_extents" > gpurun_out/st_$v.log 2>&1; echo "variant $v tests rc=$? $(tail -1 gpurun_out/st_$v.log)" >> gpurun_out/stages.log
  for zc in 32 64 128; do
    SF_SWEEP_VARIANT=$v SF_ZC=$zc timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vb.log 2>&1
    python -c "
import json
l=[x for x in open('gpurun_out/vb.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('variant $v zc $zc', (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons']) if d else open('gpurun_out/vb.log').read()[-300:])
" >> gpurun_out/stages.log
  done
done
