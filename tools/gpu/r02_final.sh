#!/bin/bash
# round 2, final 1-GPU validation: the whole GPU suite, smoke(), the C3 bench (3 timed steps after
# 3 warm-ups) and the launch list of one timed solve
mkdir -p gpurun_out/r02f
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02f/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r02f/pytest.log | tail -8
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02f/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02f/smoke.log
timeout 2400 python bench.py --steps 3 --warmup 3 > gpurun_out/r02f/bench_c3_n1.json 2> gpurun_out/r02f/bench_c3_n1.err; echo "bench rc=$?"
grep "^{" gpurun_out/r02f/bench_c3_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'], d['cpu_baseline']['value'], d['clocks'])"
BSE200_PROFILE_RANGE=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/r02f/ncu_launch.log 2>&1; echo "ncu rc=$?"
python tools/ncu_shares.py gpurun_out/r02f/launches.csv > gpurun_out/r02f/launch_shares.txt 2>&1; head -12 gpurun_out/r02f/launch_shares.txt
