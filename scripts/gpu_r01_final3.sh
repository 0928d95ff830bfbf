# round-end check: full GPU suite, smoke, default bench line, configs[4] default lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_full.log)"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? $(grep '^{' gpurun_out/bench_default.json | cut -c1-200)"
for r in 2 3; do timeout 300 python bench.py --workload stencil --radius $r > gpurun_out/c5_default_r$r.json 2>&1; echo "c5 r$r rc=$? $(grep '^{' gpurun_out/c5_default_r$r.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["roofline"]["avg_launch_ms"], d["roofline"]["frac"])')"; done
