#!/bin/bash
# 4 GPUs: dist_check (NCCL, real-split filter + RR on the tiles), C3 bench at N = 4 and N = 2
mkdir -p gpurun_out
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544"
timeout 600 $TR4 tools/dist_check.py > gpurun_out/r63_dist_check_n4.log 2>&1; echo "dist_check n4 rc=$?"; grep "world" gpurun_out/r63_dist_check_n4.log | tail -10
for NG in 4 2; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 2955$NG"
timeout 1200 $TR bench.py --gpus $NG > gpurun_out/r63_bench_c3_n$NG.json 2> gpurun_out/r63_bench_c3_n$NG.err; echo "bench n$NG rc=$?"
grep "^{" gpurun_out/r63_bench_c3_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], d['filter_algorithm'], d['roofline']['achieved'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'], repr(s['lambda_1']))"
done
