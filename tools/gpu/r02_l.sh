#!/bin/bash
# round 2, call l (1 GPU): every GPU test incl. C3 parity against the reference's own C3 solve,
# the default bench line (parity_vs_reference at C3), smoke
mkdir -p gpurun_out/r02l
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02l/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r02l/pytest.log | tail -8
timeout 300 python __graft_entry__.py > gpurun_out/r02l/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02l/smoke.log
timeout 2400 python bench.py --steps 3 --warmup 1 > gpurun_out/r02l/bench_c3.json 2> gpurun_out/r02l/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02l/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d.get('cpu_baseline',{}).get('value')); print(json.dumps(d['parity_vs_reference']))"
