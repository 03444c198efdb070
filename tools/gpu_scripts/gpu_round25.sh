#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x -k "mixed" > gpurun_out/pytest_mixed.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_mixed.log
for cfg in c2 c3; do
BSE200_MIXED=1 timeout 900 python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu > gpurun_out/b25_$cfg.json 2> gpurun_out/b25_$cfg.err; echo "$cfg rc=$?"
grep "^{" gpurun_out/b25_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['solve']['locked_per_iter'], d['solve']['filter_precision_per_iter'], d['solve']['lambda_1'], d['solve']['lambda_nev'], d['solve']['max_residual'])"
done
