for pf in 0 1 2 3 4 0; do
  SF_S2_PF=$pf timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf=$pf', d['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
