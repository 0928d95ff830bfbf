# Round-end evidence (run under gpurun, one GPU): GPU suite, smoke(), the bench
# lines committed under profiles/r02_*. The ncu capture is scripts/gpu_r02_ncu_pass.sh.
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02_smoke.log
# configs[1] 512^3 fp64 (the driver's command), then configs[3] on one GPU, fp32, configs[0]
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
timeout 900 python bench.py --strong 1024 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_strong1024.json 2> gpurun_out/r02_bench_strong1024.err
timeout 900 python bench.py --dtype f32 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench_f32.json 2> gpurun_out/r02_bench_f32.err
timeout 900 python bench.py --config c0 --steps 100 --warmup 3 > gpurun_out/r02_bench_c0.json 2> gpurun_out/r02_bench_c0.err
