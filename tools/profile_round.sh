#!/bin/bash
# Round profile captures (run on the GPU box from the repo root; then, here,
# `python tools/summarize_profiles.py <tag> 6` writes the profiles/ summaries):
#   launch list of one eager C3 step (bench.py --no-graph --no-cpu --no-e2e runs 6 eager steps),
#   ncu --set full of the dominant kernel and of the other hot-path kernels,
#   ncu --set full of one multi-CTA exact BK panel on the pivot-heavy C5 matrix.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-graph --no-cpu --no-e2e --no-scopf --no-ipm"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    $B > gpurun_out/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_tma --launch-skip 10 --launch-count 1 \
    -o gpurun_out/upd_full -f $B > /dev/null 2>&1
ncu -i gpurun_out/upd_full.ncu-rep --page raw --csv > gpurun_out/upd_full_raw.csv
ncu --set full --clock-control none \
    -k regex:"k_panel_diag|k_panel_trsm|k_panel_exact|k_panel_fast|k_trsv_fwd|k_trsv_bwd|k_step_vectors" \
    --launch-count 12 -o gpurun_out/misc_full -f $B > /dev/null 2>&1
ncu -i gpurun_out/misc_full.ncu-rep --page raw --csv > gpurun_out/misc_full_raw.csv
timeout 900 ncu --set full --clock-control none -k regex:k_panel_exact --launch-skip 200 --launch-count 1 \
    -o gpurun_out/exact_full -f python bench.py --config C5 --steps 1 --warmup 0 --no-cpu --no-e2e --no-scopf --no-ipm > /dev/null 2>&1
ncu -i gpurun_out/exact_full.ncu-rep --page raw --csv > gpurun_out/exact_full_raw.csv
ncu --set full --clock-control none -k regex:"k_step_vectors|k_trsv_fwd|k_trsv_bwd|k_recover|k_inv_blocks|k_gather|k_dsolve" \
    --launch-count 7 -o gpurun_out/solve_full -f $B > /dev/null 2>&1
ncu -i gpurun_out/solve_full.ncu-rep --page raw --csv > gpurun_out/solve_full_raw.csv
# condensation kernels of one C3 step
ncu --set full --clock-control none -k regex:"k_condense|k_anorm" --launch-skip 8 --launch-count 4 \
    -o gpurun_out/cond_full -f python tools/yy_bench.py C3 uniform > /dev/null 2>&1
ncu -i gpurun_out/cond_full.ncu-rep --page raw --csv > gpurun_out/cond_full_raw.csv
# batched (C4-shaped, 64 scenarios): the batched update, F2 and condense tiles
OZB=64 OZ=0 ncu --set full --clock-control none -k regex:"k_update_tma|k_condense_tiles" --launch-skip 20 --launch-count 3 \
    -o gpurun_out/batched_full -f python tools/oz_prof.py > /dev/null 2>&1
ncu -i gpurun_out/batched_full.ncu-rep --page raw --csv > gpurun_out/batched_full_raw.csv
# keep the merged-back payload under gpurun's 64 MiB: the raw CSVs are what summarize_profiles reads
rm -f gpurun_out/misc_full.ncu-rep gpurun_out/exact_full.ncu-rep gpurun_out/solve_full.ncu-rep \
      gpurun_out/cond_full.ncu-rep gpurun_out/batched_full.ncu-rep
ls -la gpurun_out
