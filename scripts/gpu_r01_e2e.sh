mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "staged or async or persistent" > gpurun_out/e2e_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/e2e_tests.log)"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"
python - <<'P'
import json
l=[x for x in open("gpurun_out/bench_e2e.json") if x.startswith("{")][-1]; d=json.loads(l)
print(d.get("value"), d.get("ms_per_step"), d.get("e2e"), d.get("clocks"))
P
