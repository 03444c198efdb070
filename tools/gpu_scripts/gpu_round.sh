#!/bin/bash
# one GPU call: tests, smoke, kernel microbench (plain runs only)
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
python tools/bench_hop.py > gpurun_out/bench_hop.log 2>&1; echo "bench_hop rc=$?" >> gpurun_out/bench_hop.log
tail -30 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log gpurun_out/bench_hop.log
