#!/bin/bash
mkdir -p gpurun_out
NG=4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29591"
for CM in 512; do
BSE200_CHUNK_MIN=$CM timeout 1200 $TR bench.py --gpus $NG --no-cpu --no-e2e > gpurun_out/b54_chunk$CM.json 2> gpurun_out/b54_chunk$CM.err; echo "chunk $CM rc=$?"
grep "^{" gpurun_out/b54_chunk$CM.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['solve']['ledger_seconds'], d['solve']['locked_per_iter'])"
done
