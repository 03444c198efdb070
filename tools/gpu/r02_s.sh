#!/bin/bash
# round 2, call s (1 GPU): GPU tests, C3 bench, ncu --set full of the new default tile at C3
mkdir -p gpurun_out/r02s
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02s/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r02s/pytest.log | tail -5
timeout 2400 python bench.py --steps 3 --warmup 1 > gpurun_out/r02s/bench_c3.json 2> gpurun_out/r02s/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02s/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'])"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hop_rs_tma_kernel -c 1 -o gpurun_out/r02s/ncu_rs4_c3 python tools/rs_bench.py 20000 1200 90 > gpurun_out/r02s/ncu_rs.log 2>&1; echo "ncu full rc=$?"
BSE200_PROFILE_RANGE=1 timeout 1800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s/ncu_launches_bench_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02s/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_shares.py gpurun_out/r02s/ncu_launches_bench_c3.csv > gpurun_out/r02s/ncu_launch_shares_bench_c3.txt; head -8 gpurun_out/r02s/ncu_launch_shares_bench_c3.txt
