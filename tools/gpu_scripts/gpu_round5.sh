#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
python tools/bench_ops.py > gpurun_out/bench_ops.log 2>&1; echo "bench_ops rc=$?"; cat gpurun_out/bench_ops.log
BSE200_FILTER=3m timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c3_3m.json 2> gpurun_out/bench_c3_3m.err; echo "c3 3m rc=$?"
cat gpurun_out/bench_c3_3m.json; tail -3 gpurun_out/bench_c3_3m.err
