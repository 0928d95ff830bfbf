mkdir -p gpurun_out
: > gpurun_out/hints.log
SF_SWEEP_HINTS=3 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ten_steps or projection or odd_extents or bench128" > gpurun_out/hints_t.log 2>&1; echo "hints tests rc=$? $(tail -1 gpurun_out/hints_t.log)" >> gpurun_out/hints.log
for cfg in "0 x" "1 x" "2 x" "3 x" "0 0" "0 1" "3 1"; do
  set -- $cfg
  if [ "$2" = "x" ]; then unset SF_L2_PROMO; else export SF_L2_PROMO=$2; fi
  SF_SWEEP_HINTS=$1 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vb.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/vb.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('hints $1 promo $2', (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['power_w_max']) if d else open('gpurun_out/vb.log').read()[-300:])
" >> gpurun_out/hints.log
done
