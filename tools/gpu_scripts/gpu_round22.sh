#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/c64_diag.py > gpurun_out/c64_diag.log 2>&1; echo "rc=$?"; grep -v Warn gpurun_out/c64_diag.log
timeout 600 python -m pytest tests -q -m gpu -x -k "c64" > gpurun_out/pytest_c64.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_c64.log
