mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_executor.py -q -x > gpurun_out/zqc_tests.log 2>&1; echo "exec tests rc=$? $(tail -1 gpurun_out/zqc_tests.log)"
tail -30 gpurun_out/zqc_tests.log | grep -E "Error|error" | head -5
cp paper_1201_2118_b200/_lib/libsfb200.so /tmp/lib_orig.so
for L in orig before orig before; do
  if [ "$L" = "orig" ]; then cp /tmp/lib_orig.so paper_1201_2118_b200/_lib/libsfb200.so; else cp scripts/probes/libs/lib_$L.so paper_1201_2118_b200/_lib/libsfb200.so; fi
  touch paper_1201_2118_b200/_lib/libsfb200.so
  for r in 2 3; do
    echo -n "$L r=$r: "; timeout 300 python bench.py --workload stencil --radius $r --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}; print(d['value'], r.get('avg_launch_ms'), r.get('frac'))"
  done
done
cp /tmp/lib_orig.so paper_1201_2118_b200/_lib/libsfb200.so
