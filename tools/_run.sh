timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -1 > gpurun_out/t1.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_r1f.json 2> gpurun_out/bench_r1f.err
bash tools/profile_round.sh c3 r1f > /dev/null 2>&1
timeout 1200 python tools/sweep.py --steps 10 --tag r1f > /dev/null 2>&1; cp profiles/r1f_sweep.* gpurun_out/
cat gpurun_out/t1.txt gpurun_out/smoke.txt gpurun_out/bench_r1f.json
