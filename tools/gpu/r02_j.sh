#!/bin/bash
# round 2, call j (1 GPU): GPU tests, C4 (n = 100k) on ONE GPU with the operator held as planes only
mkdir -p gpurun_out/r02j
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02j/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/r02j/pytest.log | tail -8
timeout 2700 python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r02j/bench_c4_n1.json 2> gpurun_out/r02j/bench_c4_n1.err; echo "c4 n1 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02j/bench_c4_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['filter_algorithm'], d['roofline']['frac'], d['solve']['iterations'], d['solve']['ledger_seconds'], d['memory'], d['solve']['lambda_1'], d['solve']['locked_per_iter'])"
tail -3 gpurun_out/r02j/bench_c4_n1.err
