#!/bin/bash
mkdir -p gpurun_out
for cfg in c3b0 c3mixed c3c64; do
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --config $cfg --no-cpu > gpurun_out/b46_$cfg.json 2> gpurun_out/b46_$cfg.err; echo "$cfg rc=$?"
grep "^{" gpurun_out/b46_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']), d.get('filter_tflops_per_gpu'))"
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561"
timeout 2400 $TR bench.py --gpus 4 --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/b46_c4_n4.json 2> gpurun_out/b46_c4_n4.err; echo "c4 n4 rc=$?"
grep "^{" gpurun_out/b46_c4_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], s['ledger_seconds'], s['iterations'], s['converged'], d['filter_tflops_per_gpu'], s['locked_per_iter'])"
tail -3 gpurun_out/b46_c4_n4.err
