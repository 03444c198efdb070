#!/bin/bash
# round 2, call p (1 GPU): a 4-warp 32 x 32 warp-tile variant of the real-split kernel (2 CTAs/SM)
mkdir -p gpurun_out/r02p
timeout 900 python tools/rs_bench.py 20000 1200,600,300 90,93,95 > gpurun_out/r02p/rs_tall4.txt 2>&1; echo "rc=$?"; cat gpurun_out/r02p/rs_tall4.txt
