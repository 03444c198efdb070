#!/bin/bash
# round 2, call z (1 GPU): c64 pair kernel with column tiles fastest (clusters along y):
# c64 / split-K tests, C3 c64 bench, ncu traffic of one k ~ 1200 pair-kernel launch
mkdir -p gpurun_out/r02z
timeout 900 python -m pytest tests -m gpu -q -k "c64 or split_k" > gpurun_out/r02z/pytest_c64.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02z/pytest_c64.log
timeout 900 python bench.py --config c3c64 --steps 3 --warmup 3 --no-cpu > gpurun_out/r02z/bench_c3c64_n1.json 2> gpurun_out/r02z/bench_c3c64.err; echo "bench rc=$?"
grep "^{" gpurun_out/r02z/bench_c3c64_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['solve']['ledger_seconds'], d['roofline']['achieved'], d['clocks'])"
timeout 900 ncu --set full --clock-control none -k regex:step_kernel --launch-skip 40 -c 1 -o gpurun_out/r02z/ncu_c64_pair python bench.py --config c3c64 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/r02z/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r02z/ncu_c64_pair.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,lts__t_sector_hit_rate.pct > gpurun_out/r02z/ncu_c64_pair_raw.csv 2>&1; cat gpurun_out/r02z/ncu_c64_pair_raw.csv | head -5
