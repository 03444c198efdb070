#!/bin/bash
# round 2, call q (1 GPU): 4-warp real-split tiles, 4 vs 3 stages, both directions
mkdir -p gpurun_out/r02q
timeout 900 python tools/rs_bench.py 20000 1200,810,600 90,95,96 > gpurun_out/r02q/rs_tall4.txt 2>&1; echo "rc=$?"; cat gpurun_out/r02q/rs_tall4.txt
