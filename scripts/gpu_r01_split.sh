mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "temporal or golden or bench128 or random or moving" > gpurun_out/split_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/split_tests.log)"
AB_LIBS="orig before orig before" bash scripts/probes/ab_libs.sh
