python tools/_dbg2.py 2>&1 | tail -4
timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -2
timeout 1200 python tools/sweep.py --steps 10 --tag r1d 2>&1 | tail -1
mkdir -p gpurun_out; cp profiles/r1d_sweep.* gpurun_out/
