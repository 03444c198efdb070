#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests -q -m gpu -x -k "c64" > gpurun_out/pytest_c64.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_c64.log
