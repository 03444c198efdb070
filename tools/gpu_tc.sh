#!/bin/bash
mkdir -p gpurun_out
timeout 60 ./tools/tc_probe 256 256 512 > gpurun_out/tc_probe.log 2>&1; echo "rc=$?" >> gpurun_out/tc_probe.log
timeout 60 ./tools/tc_probe 300 200 1000 >> gpurun_out/tc_probe.log 2>&1; echo "rc=$?" >> gpurun_out/tc_probe.log
cat gpurun_out/tc_probe.log
