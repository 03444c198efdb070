#!/bin/bash
# round 2, call k (4 GPUs): C3 at N = 4 / 2 with rank-0 generation + broadcast and the two-half
# start block, NCCL parity at N = 4
mkdir -p gpurun_out/r02k
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543"
timeout 900 $TR4 tools/dist_check.py > gpurun_out/r02k/dist_check_n4.txt 2>&1; echo "dist_check4 rc=$?"
grep -cE " OK" gpurun_out/r02k/dist_check_n4.txt; grep FAIL gpurun_out/r02k/dist_check_n4.txt
for N in 4 2; do
  TR=$([ $N = 4 ] && echo "$TR4" || echo "$TR2")
  timeout 1800 $TR bench.py --gpus $N --steps 3 --warmup 1 > gpurun_out/r02k/bench_c3_n$N.json 2> gpurun_out/r02k/bench_c3_n$N.err; echo "bench n$N rc=$?"
  grep "^{" gpurun_out/r02k/bench_c3_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['generator_s'], d['memory'])"
done
