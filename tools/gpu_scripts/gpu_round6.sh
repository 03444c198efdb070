#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python tools/tune_hop.py > gpurun_out/tune_hop.log 2>&1; echo "tune rc=$?"; cat gpurun_out/tune_hop.log
