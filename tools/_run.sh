timeout 900 python -m pytest tests/test_mha_gpu.py -x -q 2>&1 | tail -1 > gpurun_out/t1.txt
python tools/time_variants.py --configs c3,c3_nc --steps 20 head 2>&1
cat gpurun_out/t1.txt
