#!/bin/bash
# FP64 peak probe on the GPU box with clock sampling.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peak_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.log 2>&1
RC=$?
kill $SMI
nvidia-smi > gpurun_out/nvidia_smi.txt
lscpu > gpurun_out/lscpu.txt; nproc >> gpurun_out/lscpu.txt
cat gpurun_out/fp64_peak.log
exit $RC
