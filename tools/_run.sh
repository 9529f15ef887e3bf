timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2 > gpurun_out/t1.txt
python tools/time_variants.py --configs c3,c3_nc,c2_4k,c4 --steps 20 head 2>&1
cat gpurun_out/t1.txt
