#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c2 --steps 1 --warmup 1 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
cat gpurun_out/bench_c2.json; tail -5 gpurun_out/bench_c2.err
timeout 1500 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
cat gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
