mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "periodic or temporal or golden" > gpurun_out/perab_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/perab_tests.log)"
timeout 300 python scripts/probes/parity_stress.py 1500 31 150 > gpurun_out/parity_perab.log 2>&1; echo "stress rc=$? $(tail -1 gpurun_out/parity_perab.log)"
AB_LIBS="orig before orig before" bash scripts/probes/ab_libs.sh
