python tools/time_variants.py --configs c2_4k,c4 --steps 20 f2 f3 k2 k0 q4 q2 2>&1
