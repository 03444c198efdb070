#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/c64_diag.py > gpurun_out/c64_diag.log 2>&1; echo "rc=$?"; cat gpurun_out/c64_diag.log | grep -v Warn
