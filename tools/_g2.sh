python tools/yy_bench.py C3 uniform 2>&1 | tail -1
python tools/yy_bench.py C3 local 2>&1 | tail -1
python tools/yy_bench.py C4 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
