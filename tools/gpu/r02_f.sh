#!/bin/bash
# round 2, call f (1 GPU): GPU tests, C3 bench (default), HBM kernels (L2 flushed), ncu launch list
# of the bench command, one ncu --set full capture of the real-split kernel at C3
mkdir -p gpurun_out/r02f
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02f/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r02f/pytest.log | tail -8
timeout 1800 python bench.py --steps 2 --warmup 1 > gpurun_out/r02f/bench_c3.json 2> gpurun_out/r02f/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02f/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['cpu_baseline']['value'], d['is_definite'])"
timeout 600 python tools/hbm_kernels.py > gpurun_out/r02f/hbm_kernels.txt 2>&1; echo "hbm rc=$?"; cat gpurun_out/r02f/hbm_kernels.txt
cp gpurun_out/hbm_kernels.json gpurun_out/r02f/ 2>/dev/null
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02f/ncu_launches_bench_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r02f/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hop_rs_tma_kernel -c 1 -o gpurun_out/r02f/ncu_rs_c3 python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02f/ncu_rs.log 2>&1; echo "ncu full rc=$?"
