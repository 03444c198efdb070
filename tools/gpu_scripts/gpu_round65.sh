#!/bin/bash
# final 1-GPU check: RS tile sweep incl. BK = 32 / 8-stage variants, full GPU suite, smoke
mkdir -p gpurun_out
timeout 600 python tools/tune_rs.py 20000 1200,300 92,95,96,94 2>&1 | tail -8 | tee gpurun_out/r65_tune_rs.txt
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r65_pytest_gpu.log; tail -3 gpurun_out/r65_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r65_smoke.log 2>&1; tail -1 gpurun_out/r65_smoke.log
