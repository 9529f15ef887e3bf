#!/usr/bin/env bash
O=gpurun_out/r2h
mkdir -p $O
timeout 900 python tools/time_variants.py --configs c3 --steps 20 base nomath nostage nowait 2>&1 | tee $O/variants.txt
