mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "persistent or golden or re100 or taylor or odd_extents or projection or smoke or harness or nan" > gpurun_out/pl2_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/pl2_tests.log)"
tail -30 gpurun_out/pl2_tests.log | grep -E "Error|error|assert" | head -10
cp paper_1201_2118_b200/_lib/libsfb200.so /tmp/lib_orig.so
for L in orig before orig before; do
  if [ "$L" = "orig" ]; then cp /tmp/lib_orig.so paper_1201_2118_b200/_lib/libsfb200.so; else cp scripts/probes/libs/lib_$L.so paper_1201_2118_b200/_lib/libsfb200.so; fi
  touch paper_1201_2118_b200/_lib/libsfb200.so
  echo -n "$L: "; timeout 300 python scripts/probes/persist_probe.py 129x129x3,64x64x64,96x96x96 2>&1 | tail -1
done
cp /tmp/lib_orig.so paper_1201_2118_b200/_lib/libsfb200.so
timeout 300 python scripts/probes/small_grid_probe.py 1 2>&1 | tail -1
