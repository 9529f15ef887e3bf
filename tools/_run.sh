python tools/time_variants.py --configs c3,c2_4k,c4 --steps 20 head 2>&1
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -1
