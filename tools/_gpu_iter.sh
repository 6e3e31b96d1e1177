set -x
python tools/yy_bench.py C3 uniform
python tools/yy_bench.py C3 local
python tools/yy_bench.py C4
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -15
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c3 or c4 or c2" 2>&1 | tail -15
python bench.py --steps 10 --warmup 3 2>&1 | tail -2 | cut -c1-1500
