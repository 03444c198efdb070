#!/bin/bash
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --config c3c64 --no-cpu > gpurun_out/b48_c3c64_n1.json 2> gpurun_out/b48_c3c64_n1.err; echo "c3c64 n1 rc=$?"
grep "^{" gpurun_out/b48_c3c64_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']))"
for NG in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2957$NG"
timeout 1200 $TR bench.py --gpus $NG --config c3c64 --no-cpu > gpurun_out/b48_c3c64_n$NG.json 2> gpurun_out/b48_c3c64_n$NG.err; echo "c3c64 n$NG rc=$?"
grep "^{" gpurun_out/b48_c3c64_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'])"
done
