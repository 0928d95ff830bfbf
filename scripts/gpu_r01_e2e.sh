mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/t_tests.log 2>&1; rc=$?
echo "tests rc=$rc $(tail -1 gpurun_out/t_tests.log)"
if [ $rc -ne 0 ]; then tail -60 gpurun_out/t_tests.log; exit 1; fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"
python -c "
import json
l=[x for x in open('gpurun_out/bench_e2e.json') if x.startswith('{')]
d=json.loads(l[-1]); print(d['value'], d['ms_per_step'], d['e2e'], d['clocks'])
"
