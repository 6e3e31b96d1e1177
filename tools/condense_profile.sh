python tools/yy_bench.py C3 uniform 2>&1 | tail -1
python tools/yy_bench.py C3 local 2>&1 | tail -1
python tools/yy_bench.py C4 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "condense or c3 or c4 or c2" 2>&1 | tail -4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_condense_tiles|k_condense_diag|k_condense_rows" -s 6 -c 3 -o gpurun_out/prof_cond python tools/yy_bench.py C3 uniform > gpurun_out/ncu_cond.log 2>&1
tail -3 gpurun_out/ncu_cond.log
