mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k_update_tma --launch-skip 10 --launch-count 1 -o gpurun_out/upd_full2 -f python bench.py --steps 1 --warmup 0 --no-graph --no-cpu --no-e2e > gpurun_out/ncu_upd.log 2>&1
ncu -i gpurun_out/upd_full2.ncu-rep --page raw --csv > gpurun_out/upd_full2_raw.csv 2>&1
ncu -i gpurun_out/upd_full2.ncu-rep --page source --csv --print-source sass > gpurun_out/upd_full2_src.csv 2>&1
ls -la gpurun_out
