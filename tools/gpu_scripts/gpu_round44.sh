#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -m gpu -k "dist or c64" 2>&1 | tail -3
for NG in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2954$NG"
timeout 600 $TR tools/dist_check.py > gpurun_out/dist_check_n$NG.log 2>&1; echo "dist_check n$NG rc=$?"; grep "world" gpurun_out/dist_check_n$NG.log | tail -10
timeout 1200 $TR bench.py --gpus $NG --config c3c64 --no-cpu > gpurun_out/b44_c3c64_n$NG.json 2> gpurun_out/b44_c3c64_n$NG.err; echo "bench c3c64 n$NG rc=$?"
grep "^{" gpurun_out/b44_c3c64_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']))"
tail -3 gpurun_out/b44_c3c64_n$NG.err
done
