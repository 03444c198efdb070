#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python bench.py --no-cpu > gpurun_out/b38_c3.json 2> gpurun_out/b38_c3.err; echo "bench rc=$?"
grep "^{" gpurun_out/b38_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['solve']['ledger_seconds'], d['solve']['iterations'])"
tail -3 gpurun_out/b38_c3.err
