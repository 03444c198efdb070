#!/bin/bash
# round 2, call h (4 GPUs): C3 at N = 1 / 2 / 4 after the start-block changes, NCCL parity at N = 4
mkdir -p gpurun_out/r02h
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR4 tools/dist_check.py > gpurun_out/r02h/dist_check_n4.txt 2>&1; echo "dist_check4 rc=$?"
grep -cE " OK" gpurun_out/r02h/dist_check_n4.txt; grep FAIL gpurun_out/r02h/dist_check_n4.txt
for N in 4 2; do
  TR=$([ $N = 4 ] && echo "$TR4" || echo "$TR2")
  timeout 1800 $TR bench.py --gpus $N --steps 3 --warmup 1 > gpurun_out/r02h/bench_c3_n$N.json 2> gpurun_out/r02h/bench_c3_n$N.err; echo "bench n$N rc=$?"
  grep "^{" gpurun_out/r02h/bench_c3_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'])"
done
timeout 1800 python bench.py --steps 3 --warmup 1 --no-cpu > gpurun_out/r02h/bench_c3_n1.json 2> gpurun_out/r02h/bench_c3_n1.err; echo "bench n1 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02h/bench_c3_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'])"
