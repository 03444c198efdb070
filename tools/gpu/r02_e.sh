#!/bin/bash
# round 2, call e: RS consumer variants (V0 stage-wise / V1 runtime-rot pipelined / V2 per-part
# pipelined / V3 round-1 generic loads) at the C3 operator size, then ncu on the best two
mkdir -p gpurun_out/r02e
timeout 900 python tools/rs_bench.py 20000 1200,300 92,101,102,103 > gpurun_out/r02e/rs_variants_tall.txt 2>&1; echo "tall rc=$?"
cat gpurun_out/r02e/rs_variants_tall.txt
timeout 900 python tools/rs_bench.py 20000 300,100 94,104,105,106 > gpurun_out/r02e/rs_variants_narrow.txt 2>&1; echo "narrow rc=$?"
cat gpurun_out/r02e/rs_variants_narrow.txt
