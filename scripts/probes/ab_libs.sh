# A/B timing of alternate builds of libsfb200.so (bench k_sweep2 launch time)
cp paper_1201_2118_b200/_lib/libsfb200.so /tmp/lib_orig.so
for L in ${AB_LIBS:-orig before orig before}; do
  if [ "$L" = "orig" ]; then cp /tmp/lib_orig.so paper_1201_2118_b200/_lib/libsfb200.so; else cp scripts/probes/libs/lib_$L.so paper_1201_2118_b200/_lib/libsfb200.so; fi
  touch paper_1201_2118_b200/_lib/libsfb200.so
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', d['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'])"
done
