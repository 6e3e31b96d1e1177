set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/yy_bench.py C3 uniform 2>&1 | tail -3
python tools/yy_bench.py C3 local 2>&1 | tail -3
python tools/yy_bench.py C4 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -2 | cut -c1-3000
