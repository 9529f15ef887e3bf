set -x
timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_r1e.json 2> gpurun_out/bench_r1e.err; cat gpurun_out/bench_r1e.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
bash tools/profile_round.sh c3 r1e > /dev/null 2>&1
timeout 1200 python tools/sweep.py --steps 10 --tag r1e > /dev/null 2>&1; cp profiles/r1e_sweep.* gpurun_out/
