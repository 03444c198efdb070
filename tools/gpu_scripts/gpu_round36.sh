#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_dist.py -q -m gpu 2>&1 | tail -1
for NG in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2952$NG"
timeout 600 $TR tools/dist_check.py > gpurun_out/dist_check_n$NG.log 2>&1; echo "dist_check n$NG rc=$?"; grep "world" gpurun_out/dist_check_n$NG.log | tail -8
timeout 1200 $TR bench.py --gpus $NG --no-cpu > gpurun_out/b36_c3_n$NG.json 2> gpurun_out/b36_c3_n$NG.err; echo "bench n$NG rc=$?"
grep "^{" gpurun_out/b36_c3_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'], d['clocks'])"
done
