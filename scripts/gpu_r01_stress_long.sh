mkdir -p gpurun_out
for sd in 101 102 103; do PS_MAXEXT=100 timeout 400 python scripts/probes/parity_stress.py 5000 $sd 300 > gpurun_out/ps_long_$sd.log 2>&1; echo "ref seed $sd rc=$? $(tail -1 gpurun_out/ps_long_$sd.log)"; grep DIFF gpurun_out/ps_long_$sd.log | head -3; done
for sd in 201 202; do timeout 300 python scripts/probes/parity_stress.py 5000 $sd 200 bc > gpurun_out/ps_bc_$sd.log 2>&1; echo "bc seed $sd rc=$? $(tail -1 gpurun_out/ps_bc_$sd.log)"; grep DIFF gpurun_out/ps_bc_$sd.log | head -3; done
for sd in 301 302; do timeout 400 python scripts/probes/executor_stress.py 5000 $sd 300 > gpurun_out/es_$sd.log 2>&1; echo "exec seed $sd rc=$? $(tail -1 gpurun_out/es_$sd.log)"; grep DIFF gpurun_out/es_$sd.log | head -3; done
