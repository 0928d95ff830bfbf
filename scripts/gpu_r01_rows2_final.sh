# default two-rows-per-thread JIT template: full GPU suite, smoke, configs[4] bench lines, ncu of the radius-2/3 kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/gpu_tests_full.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/gpu_tests_full.log)"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
for r in 2 3; do for t in 32,8,64 32,16,64; do
  timeout 300 python bench.py --workload stencil --radius $r --tile $t --steps 10 --warmup 3 > gpurun_out/c5_r${r}_${t//,/_}.json 2>&1; echo "c5 r$r $t rc=$? $(grep '^{' gpurun_out/c5_r${r}_${t//,/_}.json | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["roofline"]["avg_launch_ms"], d["roofline"]["frac"], d["clocks"])')"
done; done
for r in 2 3; do
CMD="python bench.py --workload stencil --radius $r --tile 32,16,64 --steps 2 --warmup 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sf_user_kernel -s 2 -c 1 -o gpurun_out/prof_c5_rows2_r$r $CMD > gpurun_out/ncu_c5_r$r.log 2>&1; echo "ncu r$r rc=$?"
done
