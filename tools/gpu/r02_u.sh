#!/bin/bash
# round 2, call u (1 GPU): BK = 32 double-buffered 4-warp tile; tiles at the N = 4 tile size (m = 10k)
mkdir -p gpurun_out/r02u
timeout 900 python tools/rs_bench.py 20000 1200,600 96,97 > gpurun_out/r02u/rs_k32.txt 2>&1; cat gpurun_out/r02u/rs_k32.txt
timeout 900 python tools/rs_bench.py 10000 1200,600,300 92,94,96,97 > gpurun_out/r02u/rs_m10k.txt 2>&1; cat gpurun_out/r02u/rs_m10k.txt
