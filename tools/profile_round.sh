#!/bin/bash
# Round profile captures (run on the GPU box from the repo root):
#   launch list of one eager C3 step, ncu --set full of the dominant kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-graph --ref-sample 256 > gpurun_out/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_tma --launch-skip 10 --launch-count 1 \
    -o gpurun_out/upd_full -f python bench.py --steps 1 --warmup 0 --no-graph --ref-sample 256 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:"k_condense_yy|k_panel_diag|k_trsv_fwd|k_trsv_bwd|k_panel_fast|k_panel_trsm" \
    --launch-count 8 -o gpurun_out/misc_full -f python bench.py --steps 1 --warmup 0 --no-graph --ref-sample 256 > /dev/null 2>&1
ls -la gpurun_out
