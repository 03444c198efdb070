#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for cfg in c3b0 c2; do
timeout 900 python bench.py --config $cfg --steps 1 --warmup 1 > gpurun_out/b16_$cfg.json 2> gpurun_out/b16_$cfg.err; echo "$cfg rc=$?"
grep "^{" gpurun_out/b16_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'], d['solve']['locked_per_iter'])"
tail -2 gpurun_out/b16_$cfg.err
done
