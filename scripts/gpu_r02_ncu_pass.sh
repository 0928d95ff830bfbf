# ncu evidence for the temporal pass at 512^3 (run under gpurun, one GPU):
#  1. the bench command without ncu (must exit 0 first),
#  2. the per-launch list of one bench step (gpu__time_duration, serialised, cold),
#  3. one `--set full` capture of the pass's launches (k_sweep2i interior tiles,
#     k_sweep2 z/y slabs, k_sweep2 x-slab form) after warm-up.
# Summaries: python scripts/ncu_summary.py gpurun_out/r02_prof_pass.ncu-rep --name r02_ncu_pass \
#   --json profiles/ncu_sweep2.json --algo-bytes 21474836480
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 3 --sweeps 20 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/r02_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep2 -s 60 -c 3 -o gpurun_out/r02_prof_pass \
    $CMD > gpurun_out/r02_ncu_pass.log 2>&1
echo rc=$? >> gpurun_out/r02_ncu_pass.log
