mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_uv.log 2>&1; rc=$?
echo "tests rc=$rc $(tail -1 gpurun_out/t_uv.log)"
if [ $rc -ne 0 ]; then grep -E "^E |FAILED" gpurun_out/t_uv.log | head; exit 1; fi
for e in "" "SF_NO_UV_TMA=1"; do
  env $e timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --sweeps 20 > gpurun_out/vb.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/vb.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$e', (d['value'], d['ms_per_step']) if d else open('gpurun_out/vb.log').read()[-600:])
"
done
