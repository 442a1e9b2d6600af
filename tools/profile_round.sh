#!/bin/bash
# Profiling recipe for one round (run under gpurun from the repo root):
#   1. the bench command exits 0 without ncu,
#   2. ncu launch list (every launch, device time) of the same command,
#   3. ncu --set full of the dominant kernel.
# Outputs land in gpurun_out/; summaries are copied into profiles/ by tools/ncu_summary.py.
set -u
CMD="python bench.py --steps 3 --warmup 3 --spmv-reps 10 --no-cpu-baseline --no-verify --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/prof_plain.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/prof_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_tiled -s 8 -c 1 \
    -o gpurun_out/prof_top $CMD > gpurun_out/prof_full.log 2>&1

timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_tiled -c 1 \
    -o gpurun_out/prof_cg $CMD > gpurun_out/prof_cg.log 2>&1
echo "fused cg profile done"
