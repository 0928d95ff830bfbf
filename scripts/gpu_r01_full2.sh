# full GPU suite + default bench (with e2e, cpu baseline) + single-sweep A/B + reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_full.log)"
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --variant tma1 --no-e2e --no-cpu-baseline > gpurun_out/bench_tma1.json 2> gpurun_out/bench_tma1.err; echo "tma1 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'P'
import json
for f in ("bench_default","bench_tma1","bench_ref"):
    try:
        l=[x for x in open(f"gpurun_out/{f}.json") if x.startswith("{")][-1]; d=json.loads(l)
        print(f, d.get("value"), d.get("ms_per_step"), (d.get("e2e") or {}).get("value"), (d.get("roofline") or {}).get("frac"), (d.get("cpu_baseline") or {}).get("value"), d.get("clocks"))
    except Exception as e: print(f, "ERR", e)
P
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
