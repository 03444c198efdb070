#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
for cfg in c3c64 c3mixed; do
timeout 1200 python bench.py --config $cfg --no-cpu > gpurun_out/b32_$cfg.json 2> gpurun_out/b32_$cfg.err; echo "$cfg rc=$?"
grep "^{" gpurun_out/b32_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'], d['solve']['lambda_1'], d['solve']['lambda_nev'])"
done
timeout 1200 python bench.py --impl reference > gpurun_out/b32_ref.json 2> gpurun_out/b32_ref.err; echo "ref rc=$?"; cat gpurun_out/b32_ref.json
