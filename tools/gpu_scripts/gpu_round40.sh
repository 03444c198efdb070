#!/bin/bash
mkdir -p gpurun_out
NG=4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29524"
BSE200_TIMING=1 timeout 1200 $TR bench.py --gpus $NG --no-cpu --no-e2e --warmup 1 > gpurun_out/b40_n4.json 2> gpurun_out/b40_n4.err; echo "bench n4 rc=$?"
grep "dist solve" gpurun_out/b40_n4.json gpurun_out/b40_n4.err | tail -8
grep "^{" gpurun_out/b40_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['solve']['ledger_seconds'])"
