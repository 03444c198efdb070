#!/bin/bash
mkdir -p gpurun_out
NG=${NG:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29516"
timeout 600 $TR tools/dist_check.py > gpurun_out/dist_check_$NG.log 2>&1; echo "dist_check rc=$?"
grep -E "world|Error" gpurun_out/dist_check_$NG.log | head -20
timeout 900 $TR bench.py --gpus $NG --config c3 --steps 1 --warmup 1 > gpurun_out/b11_c3_n$NG.json 2> gpurun_out/b11_c3_n$NG.err; echo "c3 n$NG rc=$?"
grep "^{" gpurun_out/b11_c3_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'])"
tail -3 gpurun_out/b11_c3_n$NG.err
