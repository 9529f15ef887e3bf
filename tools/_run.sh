timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -1
python tools/time_variants.py --configs c3,c3_fp16,c3_nc,c2_512,c2_1k,c2_2k,c2_4k,c2_8k,c2_16k,c4,c5 --steps 10 2>&1 | head -11
