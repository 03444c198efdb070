#!/bin/bash
# round 2, call c (1 GPU): C2 parity vs the reference, RR factors, the reference's own test files
# against the drop-in, the CPU model vs a measured C2 oracle solve, the reference arm at C3
mkdir -p gpurun_out/r02c
timeout 2400 python -m pytest tests -m gpu -x -q -k "large_parity or rayleigh_ritz_golden or reference_suite" > gpurun_out/r02c/pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r02c/pytest.log
cp gpurun_out/ref_suite.log gpurun_out/r02c/ 2>/dev/null; tail -5 gpurun_out/r02c/ref_suite.log
timeout 2400 python tools/cpu_model_check.py c2 > gpurun_out/r02c/cpu_model_check_c2.log 2>&1; echo "cpu_model_check rc=$?"
tail -3 gpurun_out/r02c/cpu_model_check_c2.log
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02c/ref_c3.json 2> gpurun_out/r02c/ref_c3.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/r02c/ref_c3.json; tail -3 gpurun_out/r02c/ref_c3.err
cp .bench_cache/*.json gpurun_out/r02c/ 2>/dev/null
timeout 1500 python bench.py --steps 1 --warmup 1 > gpurun_out/r02c/bench_c3.json 2> gpurun_out/r02c/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02c/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d.get('cpu_baseline'))"
