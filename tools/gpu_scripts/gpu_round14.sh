#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --config c3 --steps 1 --warmup 1 > gpurun_out/b14_c3_n1.json 2> gpurun_out/b14_c3_n1.err; echo "c3 n1 rc=$?"
grep "^{" gpurun_out/b14_c3_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'], d['filter_executed_tflops_per_gpu'], d['solve']['locked_per_iter'], d['solve']['lambda_1'], d['solve']['lambda_nev'])"
