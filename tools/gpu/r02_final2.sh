#!/bin/bash
# round 2, final 1-GPU validation after the ragged-tile change: GPU suite, smoke, C3 bench
mkdir -p gpurun_out/r02g
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02g/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r02g/pytest.log | tail -8
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02g/smoke.log
timeout 2400 python bench.py --steps 3 --warmup 3 > gpurun_out/r02g/bench_c3_n1.json 2> gpurun_out/r02g/bench_c3_n1.err; echo "bench rc=$?"
grep "^{" gpurun_out/r02g/bench_c3_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'], d['cpu_baseline']['value'], d['clocks'])"
