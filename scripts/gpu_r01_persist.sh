mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/persist_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/persist_tests.log)"
for v in "SF_PERSIST=0" "SF_PERSIST=0 SF_ZC2=128" "SF_PERSIST=1" "SF_PERSIST=1 SF_PZC=1" "SF_PERSIST=1 SF_PZC=2"; do
  env $v timeout 300 python scripts/probes/persist_probe.py 2>&1 | tail -1
done
SF_PERSIST=0 timeout 300 python scripts/probes/small_grid_probe.py 1 2>&1 | tail -1
timeout 300 python scripts/probes/small_grid_probe.py 1 2>&1 | tail -1
