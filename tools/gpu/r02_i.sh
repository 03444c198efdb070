#!/bin/bash
# round 2, call i (1 GPU): GPU tests (second-stream pencil, planes-only operator, split start
# block), C3 bench, the C3 launch list (profiler range = the timed solve), C4 on ONE GPU planes-only
mkdir -p gpurun_out/r02i
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02i/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r02i/pytest.log | tail -8
timeout 1800 python bench.py --steps 3 --warmup 1 > gpurun_out/r02i/bench_c3.json 2> gpurun_out/r02i/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02i/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d.get('cpu_baseline',{}).get('value'))"
BSE200_PROFILE_RANGE=1 timeout 1800 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i/ncu_launches_bench_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02i/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_shares.py gpurun_out/r02i/ncu_launches_bench_c3.csv > gpurun_out/r02i/ncu_launch_shares_bench_c3.txt; cat gpurun_out/r02i/ncu_launch_shares_bench_c3.txt
timeout 2400 python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r02i/bench_c4_n1.json 2> gpurun_out/r02i/bench_c4_n1.err; echo "c4 n1 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02i/bench_c4_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['filter_algorithm'], d['roofline']['frac'], d['solve']['iterations'], d['solve']['ledger_seconds'], d['memory'])"
tail -3 gpurun_out/r02i/bench_c4_n1.err
