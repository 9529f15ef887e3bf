python tools/time_variants.py --configs c2_1k,c2_4k,c4,c3 --steps 20 head 2>&1
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -1
