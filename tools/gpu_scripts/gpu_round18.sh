#!/bin/bash
mkdir -p gpurun_out
NG=${NG:-4}


TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29517"

for N in 4; do
TRN="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N"
timeout 900 $TRN bench.py --gpus $N --config c3 --steps 1 --warmup 1 > gpurun_out/b18_c3_n$N.json 2> gpurun_out/b18_c3_n$N.err; echo "c3 n$N rc=$?"
grep "^{" gpurun_out/b18_c3_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'])"
done
