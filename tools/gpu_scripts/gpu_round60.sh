#!/bin/bash
# real-split filter: parity tests, then the step-rate sweep at the C3 operator size
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "rs" 2>&1 | tail -15 > gpurun_out/r60_pytest_rs.log
tail -5 gpurun_out/r60_pytest_rs.log
timeout 900 python tools/tune_rs.py 20000 1200,600,300,100 88,91,92,93,94 2>&1 | tail -30 | tee gpurun_out/r60_tune_rs.txt
