#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu.log | head -10
timeout 1200 python bench.py --no-cpu > gpurun_out/b41_c3.json 2> gpurun_out/b41_c3.err; echo "bench rc=$?"
grep "^{" gpurun_out/b41_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['solve']['locked_per_iter'])"
for NG in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2953$NG"
timeout 1200 $TR bench.py --gpus $NG --no-cpu > gpurun_out/b41_c3_n$NG.json 2> gpurun_out/b41_c3_n$NG.err; echo "bench n$NG rc=$?"
grep "^{" gpurun_out/b41_c3_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['solve']['locked_per_iter'])"
done
