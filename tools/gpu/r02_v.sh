#!/bin/bash
# round 2, call v (1 GPU): tests, default-tile choice across shapes, C3 bench, ncu of the new tile
mkdir -p gpurun_out/r02v
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02v/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r02v/pytest.log | tail -5
timeout 900 python tools/rs_bench.py 20000 1200,810,502,300,220,100 90 > gpurun_out/r02v/rs_default_m20k.txt 2>&1; cat gpurun_out/r02v/rs_default_m20k.txt
timeout 900 python tools/rs_bench.py 10000 1200,600,300 90 > gpurun_out/r02v/rs_default_m10k.txt 2>&1; cat gpurun_out/r02v/rs_default_m10k.txt
timeout 2400 python bench.py --steps 3 --warmup 1 > gpurun_out/r02v/bench_c3.json 2> gpurun_out/r02v/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02v/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'], d['cpu_baseline']['value'])"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hop_rs_tma_kernel -c 1 -o gpurun_out/r02v/ncu_rs4k32_c3 python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02v/ncu_rs.log 2>&1; echo "ncu full rc=$?"
