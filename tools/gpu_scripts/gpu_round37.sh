#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu.log | head -10
timeout 1200 python bench.py --no-cpu > gpurun_out/b37_c3.json 2> gpurun_out/b37_c3.err; echo "bench rc=$?"
grep "^{" gpurun_out/b37_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['solve']['locked_per_iter'], d['roofline']['frac'], d['roofline']['traffic'])"
