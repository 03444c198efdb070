#!/bin/bash
# re-entry check: fresh build of the library, full GPU suite, smoke, default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r59_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r59_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r59_bench.json 2> gpurun_out/r59_bench.err
tail -3 gpurun_out/r59_pytest_gpu.log; tail -2 gpurun_out/r59_smoke.log; tail -c 600 gpurun_out/r59_bench.json
