timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/sweep.py --steps 10 --tag r1c 2>&1 | tail -3
cat profiles/r1c_sweep.md
