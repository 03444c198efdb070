#!/bin/bash
# round 2, call r (1 GPU): 4-warp 3-stage tile vs the narrow tile at the small widths of a solve
mkdir -p gpurun_out/r02r
timeout 900 python tools/rs_bench.py 20000 502,400,300,220,100,40 94,96 > gpurun_out/r02r/rs_small_k.txt 2>&1; echo "rc=$?"; cat gpurun_out/r02r/rs_small_k.txt
