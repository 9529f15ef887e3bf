timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2 > gpurun_out/t.txt
python tools/time_variants.py --configs c2_512,c2_1k,c2_4k,c2_16k,c4,c3 --steps 20 head 2>&1
cat gpurun_out/t.txt
