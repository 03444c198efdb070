#!/bin/bash
# round 2, last 1-GPU validation (final plan: split under 20 waves): GPU suite,
# smoke, kernel timing at C3 widths, C3 bench
mkdir -p gpurun_out/r02z3
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02z3/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/r02z3/pytest.log | tail -8
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z3/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02z3/smoke.log
timeout 600 python tools/rs_bench.py 20000 1200,642,220 90 > gpurun_out/r02z3/rs.jsonl 2>&1; cut -c1-150 gpurun_out/r02z3/rs.jsonl
timeout 2400 python bench.py --steps 3 --warmup 3 > gpurun_out/r02z3/bench_c3_n1.json 2> gpurun_out/r02z3/bench_c3_n1.err; echo "bench rc=$?"
grep "^{" gpurun_out/r02z3/bench_c3_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'], d['clocks'])"
