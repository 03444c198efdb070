#!/bin/bash
# round 2, call a: GPU tests, smoke, one C3 bench line (exact generator, measured CPU model)
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02a/pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/r02a/smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/r02a/smoke.log
timeout 1500 python bench.py --steps 1 --warmup 1 > gpurun_out/r02a/bench_c3.json 2> gpurun_out/r02a/bench_c3.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02a/bench_c3.json; tail -5 gpurun_out/r02a/bench_c3.err
