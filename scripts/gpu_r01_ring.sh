for e in 3 5 7 3 5 7; do
  for r in 2 3; do
    echo -n "extra=$e r=$r: "; SF_JIT_RING_EXTRA=$e timeout 300 python bench.py --workload stencil --radius $r --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d.get('roofline') or {}; print(d['value'], r.get('avg_launch_ms'), r.get('frac'))"
  done
done
