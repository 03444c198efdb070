#!/bin/bash
mkdir -p gpurun_out
NG=4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29519"
timeout 2400 $TR bench.py --gpus $NG --config c4 --steps 1 --warmup 0 --no-e2e > gpurun_out/b30_c4_n4.json 2> gpurun_out/b30_c4_n4.err; echo "c4 n4 rc=$?"
grep "^{" gpurun_out/b30_c4_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['solve']['converged'], d['filter_tflops_per_gpu'], d['solve']['locked_per_iter'], d['solve']['generator_s'])"
tail -5 gpurun_out/b30_c4_n4.err
